# k_step time and replays along the developed flow of the bench slab
for w in 3 50 100 150 200 300 400 600; do timeout 300 python tools/dev_step.py $w 2>&1 | grep "^warm"; done

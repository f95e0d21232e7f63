"""Attribute ncu per-instruction samples / executed counts of k_step to the
phase of the step kernel they were inlined into (outermost wb_step.cu line),
by joining the ncu source page (cuda,sass CSV) with `nvdisasm -gi` of the
same binary.  python tools/ncu_phases.py mix.csv alli.dis [kernel-mangled-name]"""
import csv
import re
import sys

PHASES = [  # (first line, last line, name) in wb_step.cu, filled from markers
]


def phase_table(src):
    marks = []
    for i, l in enumerate(open(src), 1):
        m = re.search(r"// ---- (\([a-e]\)[^-]*|roll[^-]*|fused detection[^-]*|dt for this step)", l)
        if m:
            marks.append((i, m.group(1).strip()[:40]))
    return marks


def main(mix, dis, name, src):
    marks = phase_table(src)
    L = open(dis).read().split("\n")
    i0 = [i for i, l in enumerate(L) if l == ".text." + name + ":"][0]
    addr_ctx = {}
    block, prev_c = [], False
    sub = None
    for l in L[i0 + 1:]:
        if l.startswith(".text."):
            break
        if l.startswith("$" + name + "$"):
            sub = l.split("$")[2][:30]
            continue
        if "//## File" in l:
            if not prev_c:
                block = []
            block.append(l)
            prev_c = True
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            prev_c = False
            outer = None
            for b in block:
                for mm in re.finditer(r'wb_step\.cu", line (\d+)', b):
                    v = int(mm.group(1))
                    if v >= 540:
                        outer = v
            if sub:
                ph = "safe:" + sub
            elif outer is None:
                ph = "?"
            else:
                ph = "pre"
                for ln, nm in marks:
                    if ln <= outer:
                        ph = nm
            addr_ctx[int(m.group(1), 16)] = ph
    rows = list(csv.reader(open(mix)))
    base = None
    acc = {}
    for r in rows:
        if len(r) > 7 and r[2].startswith("0x"):
            a = int(r[2], 16)
            if base is None:
                base = a
            off = a - base
            ph = addr_ctx.get(off, "unmapped")
            s = int(r[4]) if r[4].isdigit() else 0
            ex = int(r[7]) if r[7].isdigit() else 0
            x = acc.setdefault(ph, [0, 0])
            x[0] += s
            x[1] += ex
    ts = sum(v[0] for v in acc.values()) or 1
    te = sum(v[1] for v in acc.values()) or 1
    for k, v in sorted(acc.items(), key=lambda x: -x[1][0]):
        print(f"{k:42s} samples {100*v[0]/ts:5.1f}%  warp-inst {100*v[1]/te:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2],
         sys.argv[3] if len(sys.argv) > 3 else
         "_ZN2wb6k_stepILi64ELi1ELb1ELb0EEEvNS_3GeoENS_4BufsENS_4PhysEiNS_3DbgE",
         sys.argv[4] if len(sys.argv) > 4 else "paper_1806_04960_b200/csrc/wb_step.cu")

"""Aggregate ncu --page source --print-source cuda,sass CSV into per-line
stall samples and executed instructions (top N lines)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur = None
    hdr = None
    out = []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0].isdigit() or r[2] != "-":
            continue
        samp = int(r[4]) if r[4].isdigit() else 0
        ni = int(r[5]) if r[5].isdigit() else 0
        ex = int(r[7]) if r[7].isdigit() else 0
        out.append((samp, ni, ex, cur, int(r[0]), r[1][:90]))
    tot = sum(o[0] for o in out) or 1
    totx = sum(o[2] for o in out) or 1
    print(f"total samples {tot}, warp instructions {totx}")
    for o in sorted(out, reverse=True)[:top]:
        print(f"{100*o[0]/tot:5.1f}% smp {100*o[2]/totx:5.1f}% ins  {o[3]}:{o[4]}  {o[5]}")
    by = {}
    for o in out:
        k = o[3]
        by[k] = by.get(k, 0) + o[0]
    print(by)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

"""Per-phase profile of the step kernel: joins the ncu source page of one
k_step capture (per-SASS-instruction executed counts and stall samples) with
`nvdisasm -gi` of the SAME binary (inline chains), and attributes every
instruction to the phase of step_body it was inlined into (the outermost
wb_step.cu line inside step_body, bucketed by the "// ---- (x) ..." markers).

  ncu -i rep --page source --csv --print-source cuda,sass > mix.csv
  cuobjdump -xelf all libwbflow_b200.so && nvdisasm -gi wb_capi.sm_100a.cubin > k.dis
  python tools/ncu_phases.py mix.csv k.dis

Prints a markdown table.  Fails if the SASS of the capture and of the
disassembly differ (a stale binary)."""
import csv
import re
import sys

KERNEL = ("_ZN2wb6k_stepILi128ELi3ELb1ELb0EEEvNS_3GeoENS_4BufsENS_4PhysEiNS_3DbgENS_4PartE"
          "14CUtensorMap_stS6_")  # the default launch on large grids
SRC = "paper_1806_04960_b200/csrc/wb_step.cu"


def body_range(src):
    lines = open(src).read().split("\n")
    b0 = next(i for i, l in enumerate(lines, 1) if "void step_body(" in l)
    b1 = next(i for i in range(b0, len(lines) + 1) if lines[i - 1] == "}")
    marks = []
    for i, l in enumerate(lines, 1):
        m = re.search(r"// ---- (.*?) ----", l)
        if m and b0 <= i <= b1:
            marks.append((i, m.group(1)[:34]))
    return b0, b1, marks


def disasm(dis, name):
    L = open(dis).read().split("\n")
    i0 = L.index(".text." + name + ":")
    out, block, prev, sub = [], [], False, None
    for l in L[i0 + 1:]:
        if l.startswith(".text."):
            break
        if l.startswith("$" + name + "$"):
            sub = l.split("$")[2][:40]
            continue
        if "//## File" in l:
            if not prev:
                block = []
            block.append(l)
            prev = True
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            prev = False
            chain = [(f.split("/")[-1], int(n)) for f, n in
                     re.findall(r'File "([^"]+)", line (\d+)', " ".join(block))]
            out.append((int(m.group(1), 16), m.group(2).split()[0], chain, sub))
    return out


def main(mix, dis, name=KERNEL, src=SRC):
    b0, b1, marks = body_range(src)
    out = disasm(dis, name)
    rows = list(csv.reader(open(mix)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    sidx = [i for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
    addr = {}
    for r in rows:
        if len(r) > 8 and r[2].startswith("0x"):
            addr[int(r[2], 16)] = (r[3].strip().split()[0] if r[3].strip() else "",
                                   int(r[4]) if r[4].isdigit() else 0,
                                   int(r[7]) if r[7].isdigit() else 0,
                                   int(r[8]) if r[8].isdigit() else 0,
                                   {hdr[i]: int(r[i]) for i in sidx if r[i].isdigit()})
    base = min(addr)
    bad = sum(1 for off, op, _, _ in out if addr.get(base + off, ("?",))[0] != op)
    if bad:
        sys.exit(f"{bad} SASS mismatches: the disassembly is not of the captured binary")
    acc = {}
    for off, op, chain, sub in out:
        _, s, e, th, st = addr[base + off]
        if sub:
            ph = "exact replays (out of line)"
        else:
            inner = [n for f, n in chain if f == "wb_step.cu" and b0 < n < b1]
            ph = "other"
            if inner:
                ph = "prologue"
                for ln, nm in marks:
                    if ln <= inner[-1]:
                        ph = nm
        x = acc.setdefault(ph, [0, 0, 0, {}, 0])
        x[4] += 1  # static SASS size (16 B per instruction)
        x[0] += s
        x[1] += e
        x[2] += th
        for k, v in st.items():
            x[3][k] = x[3].get(k, 0) + v
    ts = sum(v[0] for v in acc.values()) or 1
    te = sum(v[1] for v in acc.values()) or 1
    print("| phase | code KB | warp-instructions | stall samples | threads/instr | top stall reasons |")
    print("|---|---|---|---|---|---|")
    for k, v in sorted(acc.items(), key=lambda x: -x[1][0]):
        top = sorted(v[3].items(), key=lambda x: -x[1])[:3]
        tops = ", ".join(f"{n[6:]} {100 * c / max(1, v[0]):.0f}%" for n, c in top)
        print(f"| {k} | {v[4] * 16 / 1024:.1f} | {100 * v[1] / te:.1f}% | {100 * v[0] / ts:.1f}% | "
              f"{v[2] / max(1, v[1]):.1f} | {tops} |")


if __name__ == "__main__":
    main(*sys.argv[1:])

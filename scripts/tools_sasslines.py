"""Attribute ncu per-SASS metrics (--page source --print-source sass --csv)
to CUDA source lines using nvdisasm -gi line info of the same build.
usage: tools_sasslines.py <ncu_sass.csv> <disasm_gi.sass> <mangled kernel> <kernel file> <body line>
                          [region=lo-hi ...]
Each instruction is charged to the innermost location inside the kernel body
(lines >= body line of <kernel file>), following 'inlined at' chains."""
import csv, re, sys, collections

def main(csvp, sassp, fn, kfile, body, *regions):
    body = int(body)
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed"); st = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    met = {int(r[0], 16) - base: (int(r[ie] or 0), int(r[st] or 0)) for r in data}
    lines = {}
    cur = 0; infn = False
    pat = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    for l in open(sassp):
        if l.startswith(".text."):
            infn = l.strip().rstrip(":") == ".text." + fn
            continue
        if not infn:
            continue
        m = pat.search(l)
        if m:
            f1, l1, f2, l2 = m.group(1), int(m.group(2)), m.group(3), m.group(4)
            if f1.endswith(kfile) and l1 >= body:
                cur = l1
            elif f2 and f2.endswith(kfile) and int(l2) >= body:
                cur = int(l2)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            lines[int(m.group(1), 16)] = cur
    agg = collections.Counter(); sta = collections.Counter()
    for off, (c, s) in met.items():
        k = lines.get(off, -1)
        agg[k] += c; sta[k] += s
    tot = sum(agg.values()); tst = sum(sta.values())
    print(f"total warp-instr {tot:,}  stall samples {tst:,}")
    regs = []
    for r in regions:
        name, rng = r.split("=")
        lo, hi = map(int, rng.split("-"))
        regs.append((name, lo, hi))
    ra = collections.Counter(); rs = collections.Counter()
    for k in agg:
        nm = next((n for n, lo, hi in regs if lo <= k <= hi), "other")
        ra[nm] += agg[k]; rs[nm] += sta[k]
    for nm, v in ra.most_common():
        print(f"  {nm:10s} instr {v:>12,} {100*v/tot:5.1f}%   stalls {100*rs[nm]/max(tst,1):5.1f}%")
    for k, v in agg.most_common(40):
        print(f"  line {k:<5} instr {v:>12,} {100*v/tot:5.1f}%  stalls {100*sta[k]/max(tst,1):5.1f}%")

if __name__ == "__main__":
    main(*sys.argv[1:])

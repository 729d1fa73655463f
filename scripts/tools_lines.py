"""Executed warp-instructions and stall samples per source line of the tile
function, from an ncu SASS source CSV (--page source --print-source sass)
and nvdisasm -gi of the same cubin.
usage: tools_lines.py <sass.csv> <disasm_gi.sass> <mangled kernel> <call line> [name=lo-hi ...]
Each instruction is charged to the line of smol_tile (the function inlined at
<call line> of the kernel) it belongs to."""
import csv, re, sys, collections


def offsets_to_lines(sassp, fn, top):
    lines, cur, prev_hash, infn = {}, -1, False, False
    for l in open(sassp):
        if l.startswith(".text."):
            infn = l.strip().rstrip(":") == ".text." + fn
            continue
        if not infn:
            continue
        s = l.strip()
        if s.startswith("//##"):
            m = re.search(r"line (\d+) inlined at .*line (\d+)$", s)
            if m and int(m.group(2)) == top:
                cur = int(m.group(1))
            elif not prev_hash and not m:
                m2 = re.search(r"line (\d+)$", s)
                if m2:
                    cur = int(m2.group(1))
            prev_hash = True
            continue
        prev_hash = False
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            lines[int(m.group(1), 16)] = cur
    return lines


def main(csvp, sassp, fn, top, *regions):
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed"); st = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    lines = offsets_to_lines(sassp, fn, int(top))
    agg, sta, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for r in data:
        off = int(r[0], 16) - base
        k = lines.get(off, -1)
        c, s = int(r[ie] or 0), int(r[st] or 0)
        agg[k] += c; sta[k] += s
        t = r[1].split()
        op = (t[1] if t and t[0].startswith("@") else t[0]).split(".")[0] if t else "?"
        ops[k][op] += c
    tot, tst = sum(agg.values()), sum(sta.values())
    print(f"total warp-instr {tot:,}  stall samples {tst:,}")
    regs = []
    for r in regions:
        name, rng = r.split("=")
        lo, hi = map(int, rng.split("-"))
        regs.append((name, lo, hi))
    ra, rs, rop = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for k in agg:
        nm = next((n for n, lo, hi in regs if lo <= k <= hi), "other")
        ra[nm] += agg[k]; rs[nm] += sta[k]; rop[nm].update(ops[k])
    for nm, v in ra.most_common():
        print(f"  {nm:10s} instr {v:>12,} {100*v/tot:5.1f}%   stalls {100*rs[nm]/max(tst,1):5.1f}%")
        print("      ", ", ".join(f"{o} {100*c/max(v,1):.0f}%" for o, c in rop[nm].most_common(12)))
    for k, v in agg.most_common(30):
        print(f"  line {k:<5} instr {v:>12,} {100*v/tot:5.1f}%  stalls {100*sta[k]/max(tst,1):5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])

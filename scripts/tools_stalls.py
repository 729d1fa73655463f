"""Top SASS instructions by a stall reason from an ncu --page source
--print-source sass --csv dump.  usage: tools_stalls.py <csv> <reason> [n]"""
import csv, sys

def main(p, reason, n=25):
    rows = list(csv.reader(open(p))); hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    k = hdr.index(reason); ie = hdr.index("Instructions Executed")
    tot = sum(int(r[k] or 0) for r in data)
    print(f"{reason}: {tot} samples")
    for r in sorted(data, key=lambda r: -int(r[k] or 0))[:int(n)]:
        print(f"  {int(r[0],16)-base:#07x} {int(r[k] or 0):6d}  exec {int(r[ie] or 0):>9,}  {r[1].strip()[:70]}")

if __name__ == "__main__":
    main(*sys.argv[1:])

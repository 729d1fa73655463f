"""List local-memory (spill) instructions of one kernel with the kernel-body
source line they belong to.  usage: tools_spills.py <disasm -gi> <mangled> <file> <body line>"""
import re, sys

def main(sass, fn, kfile, body):
    body = int(body); cur = 0; infn = False
    pat = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    for l in open(sass):
        if l.startswith(".text."):
            infn = l.strip().rstrip(":") == ".text." + fn; continue
        if not infn: continue
        m = pat.search(l)
        if m:
            f1, l1, f2, l2 = m.group(1), int(m.group(2)), m.group(3), m.group(4)
            if f1.endswith(kfile) and l1 >= body: cur = l1
            elif f2 and f2.endswith(kfile) and int(l2) >= body: cur = int(l2)
            continue
        if "LDL" in l or "STL" in l:
            print(f"line {cur:5d}: {l.strip()[:90]}")

if __name__ == "__main__":
    main(*sys.argv[1:])

"""Update profiles/traffic.json from the ncu summaries of gpu_final_prof.sh:
DRAM read/write bytes and warp instructions per launch of each config's main
kernel.  usage: update_traffic.py <dir with ncu_<cfg>_summary.txt> <tag>"""
import json, os, sys

d, tag = sys.argv[1], sys.argv[2]
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
t = json.load(open(p))
units = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
for cfg, lay in (("c2", "dense"), ("c3a", "packed"), ("c3b", "packed"), ("c4", "packed"), ("c5", "packed")):
    f = os.path.join(d, f"ncu_{cfg}_summary.txt")
    if not os.path.exists(f):
        continue
    vals = {}
    for line in open(f):
        parts = line.split()
        if len(parts) >= 2:
            vals[parts[0]] = (parts[1], parts[2] if len(parts) > 2 else "")
    try:
        rd = float(vals["dram__bytes_read.sum"][0]) * units.get(vals["dram__bytes_read.sum"][1], 1.0)
        wr = float(vals["dram__bytes_write.sum"][0]) * units.get(vals["dram__bytes_write.sum"][1], 1.0)
        wi = float(vals["smsp__inst_executed.sum"][0])
    except (KeyError, ValueError):
        continue
    e = t.setdefault(f"{cfg}/{lay}", {})
    e.update({"read": int(rd), "write": int(wr), "warp_instr": int(wi),
              "source": f"profiles/{tag}_ncu_{cfg}_summary.txt (ncu --set full, {tag})",
              "warp_instr_source": f"profiles/{tag}_ncu_{cfg}_summary.txt (smsp__inst_executed.sum)"})
json.dump(t, open(p, "w"), indent=1)
print("updated", p)

"""Summarise an ncu report: key raw metrics + per-region (BAR.SYNC-split) instruction/stall shares."""
import csv, subprocess, sys
from collections import Counter

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))

def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    return hdr, [r for r in rows[2:] if len(r) >= len(hdr)]

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'sm__cycles_elapsed.avg.per_second',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'local_load', 'l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum']

def main(rep):
    d, u = raw(rep)
    for k in KEYS:
        if k in d:
            print(f"{k:60s} {d[k]:>16s} {u[k]}")
    for k in sorted(d):
        if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
            try:
                if float(d[k]) > 0.3:
                    print(f"{k:60s} {d[k]:>16s}")
            except ValueError:
                pass
    hdr, lines = sass(rep)
    ix = hdr.index('Instructions Executed'); isrc = hdr.index('Source')
    ist = hdr.index('Warp Stall Sampling (All Samples)')
    cols = [c for c in hdr if c.startswith('stall_') and 'Not Issued' not in c]
    tot = sum(float(r[ix] or 0) for r in lines); tst = sum(float(r[ist] or 0) for r in lines)
    bars = [i for i, r in enumerate(lines) if 'BAR.SYNC' in r[isrc]]
    prev = 0
    for b in bars + [len(lines) - 1]:
        seg = lines[prev:b + 1]
        n = sum(float(r[ix] or 0) for r in seg); st = sum(float(r[ist] or 0) for r in seg)
        sc = Counter()
        for r in seg:
            for c in cols:
                try: sc[c] += float(r[hdr.index(c)] or 0)
                except ValueError: pass
        tops = ", ".join(f"{c[6:]} {v / max(1, sum(sc.values())) * 100:.0f}%" for c, v in sc.most_common(4))
        print(f"  region [{prev}:{b}] instr {n / tot * 100:5.1f}% ({n:.3e})  stall-samples {st / tst * 100:5.1f}%  [{tops}]")
        prev = b + 1

if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise one kernel of an ncu --set full report into markdown (for profiles/).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep "title" > profiles/rNN_x.md
"""
import csv
import re
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
KEYS = [
    ("Kernel Name", "kernel"), ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_ideal.sum", "smem wavefronts (ideal)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
]
print(f"# {title}\n")
for r in rows[2:]:
    d = dict(zip(h, r))
    un = dict(zip(h, u))
    print("| metric | value |\n|---|---|")
    for k, name in KEYS:
        if k in d:
            print(f"| {name} (`{k}`) | {d[k]} {un.get(k, '')} |")
    stalls = {k: d[k] for k in h if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k) and not k.endswith("not_issued") and d[k] not in ("", "0")}
    if stalls:
        tot = sum(float(v.replace(",", "")) for v in stalls.values())
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "")))[:8]
        print("\nStall samples (top 8):\n")
        for k, v in top:
            print(f"* {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * float(v.replace(',', '')) / tot:.1f}%")
    print()

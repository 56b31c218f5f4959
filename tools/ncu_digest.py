"""Digest an ncu report: per kernel the key throughput metrics, smem wavefronts
and bank conflicts, instruction mix and the stall breakdown.
    python tools/ncu_digest.py report.ncu-rep [kernel-regex]"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "local_load", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
ST = "smsp__average_warps_issue_stalled_"
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if not re.search(kre, name):
        continue
    print("==", name[:90])
    for w in want:
        for i, c in enumerate(h):
            if c == w or (w == "local_load" and c.startswith("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum")):
                print(f"   {c}: {r[i]} {rows[1][i]}")
    st = sorted(((float(r[i] or 0), h[i][len(ST):].replace("_per_issue_active.ratio", "")) for i, c in enumerate(h)
                 if c.startswith(ST) and c.endswith("_per_issue_active.ratio")), reverse=True)[:6]
    print("   stalls:", [(round(v, 2), n) for v, n in st])

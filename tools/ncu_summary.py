"""Summarise an ncu report: key metrics + stall reasons per kernel."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
keys = {"gpu__time_duration.sum": "duration", "sm__cycles_elapsed.avg": "cycles",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy%",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
        "smsp__inst_executed.sum": "inst_executed",
        "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "lts__t_bytes.sum": "l2_bytes", "launch__registers_per_thread": "regs",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe%",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe%",
        "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex%",
        "launch__grid_size": "grid", "launch__block_size": "block"}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "?")[:60]
    print("==", name)
    for k, lab in keys.items():
        if k in d:
            print(f"   {lab:22s} {d[k]}")
    st = {h: d[h] for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
    top = sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:7]
    print("   stalls:", ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={float(v):.2f}" for k, v in top))

"""Key metrics of every kernel in an .ncu-rep (raw page), as a markdown table per kernel."""
import csv, subprocess, sys
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"] + [
        f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in
        ("long_scoreboard", "short_scoreboard", "math_pipe_throttle", "mio_throttle", "wait", "lg_throttle",
         "no_instruction", "barrier", "dispatch_stall", "not_selected", "branch_resolving", "drain", "imc_miss")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name")
for r in rows[2:]:
    print(f"\n## {r[ki][:70]}\n\n| metric | value | unit |\n|---|---|---|")
    for w in WANT:
        if w in hdr:
            print(f"| {w} | {r[hdr.index(w)]} | {units[hdr.index(w)]} |")

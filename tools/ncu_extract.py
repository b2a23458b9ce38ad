"""Write the judged metrics of one kernel from an ncu report as `name: value unit`
lines (the format bench.py's roofline.traffic reader and profiles/ use)."""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
header = sys.argv[3] if len(sys.argv) > 3 else ""
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__grid_size", "launch__cluster_dim_x",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.max.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.max.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.max.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
        "sm__ops_path_tensor_src_fp64.sum",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.max.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
names, units, vals = rows[0], rows[1], rows[2:]
with open(out, "w") as f:
    if header:
        f.write(header.rstrip() + "\n")
    for v in vals:
        f.write(f"Kernel Name: {v[names.index('Kernel Name')]}\n")
        for w in WANT:
            if w in names:
                i = names.index(w)
                f.write(f"{w}: {v[i]} {units[i]}\n")
print(open(out).read())

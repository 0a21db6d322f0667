"""Key metrics of an `ncu --set full` report (one row per profiled launch)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", "kernel"), ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_rt_%"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tmem/tensor_mem_%"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "hmma_pipe_%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data"
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        lines.append(f"== {path}")
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"  {name:22s} {r[i]} {units[i]}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))

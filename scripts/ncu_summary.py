"""Summarise one kernel of an ncu --set full report into the key metrics we cite.

    python scripts/ncu_summary.py gpurun_out/prof_philox.ncu-rep "header line" > profiles/xxx.txt
"""

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "ms"),
    ("sm__cycles_elapsed.avg", "cycle"),
    ("smsp__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__inst_executed_pipe_tex.avg.pct_of_peak_sustained_active", "%"),
    ("dram__bytes_read.sum", "byte"),
    ("dram__bytes_write.sum", "byte"),
    ("lts__t_sectors.sum", "sector"),
    ("lts__t_sectors.sum.per_second", "sector/ns"),
    ("lts__t_sectors_srcunit_tex.sum", "sector"),
    ("lts__t_sector_hit_rate.pct", "%"),
    ("l1tex__t_sectors_pipe_tex_mem_texture.sum", "sector"),
    ("l1tex__t_requests_pipe_tex_mem_texture.sum", ""),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "inst"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "inst"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "inst"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "inst"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "inst"),
    ("smsp__warps_eligible.avg.per_cycle_active", "warp"),
    ("launch__registers_per_thread", "register/thread"),
    ("launch__grid_size", ""),
    ("launch__block_size", ""),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
]


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    print(f"# {header}")
    print(f"# kernel: {v[h.index('Kernel Name')]}")
    for k, _ in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k} [{units[i]}] = {v[i]}")
    if "lts__t_sectors.sum.per_second" in h:  # derived: L2 throughput in GB/s (32-byte sectors)
        i = h.index("lts__t_sectors.sum.per_second")
        scale = {"sector/ns": 1e9, "sector/us": 1e6, "sector/ms": 1e3, "sector/s": 1.0}.get(units[i], float("nan"))
        print(f"derived: L2 sector throughput [GB/s] = {float(v[i]) * scale * 32 / 1e9:.1f}")


if __name__ == "__main__":
    main()

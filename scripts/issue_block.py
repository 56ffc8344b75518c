"""Issue and traffic summary of the Megopolis kernel from ncu --set full reports (bench.py's
``roofline.issue`` block and ``roofline.traffic``).

    python scripts/issue_block.py philox@16777216@354=gpurun_out/prof_philox.ncu-rep \
        megores@16777216@354=gpurun_out/prof_megores.ncu-rep > profiles/megopolis_issue.json

Entries are keyed "<stream>@<N>" (N the particles of the profiled launch, B its rounds).

Per stream: warp-instructions per warp-round (N*B/32 warp-rounds: one partner comparison per
lane), issue-active %, the time the kernel would take at one warp-instruction per cycle on
every SMSP (4 per SM, 148 SMs, at the measured SM clock), the kernel's fraction of that issue
roofline, the top stall reasons, and DRAM / L2 traffic per launch.
"""

import argparse
import csv
import io
import json
import subprocess


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (v[i], units[i]) for i, k in enumerate(h)}


def num(d, k, scale_units=None):
    val, unit = d[k]
    x = float(val.replace(",", ""))
    if scale_units:
        x *= scale_units.get(unit, 1.0)
    return x


def block(rep, n, b):
    d = raw(rep)
    t_s = num(d, "gpu__time_duration.sum", {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0})
    cyc = num(d, "sm__cycles_elapsed.avg")
    inst = num(d, "smsp__inst_executed.sum")
    sms = int(num(d, "device__attribute_multiprocessor_count")) if "device__attribute_multiprocessor_count" in d else 148
    clk = cyc / t_s
    t_full = inst / (sms * 4) / clk
    rounds = n * b / 32
    byte = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = num(d, "dram__bytes_read.sum", byte) + num(d, "dram__bytes_write.sum", byte)
    stalls = {}
    for k in d:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = num(d, k)
    top = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
    out = {
        "kernel": d["Kernel Name"][0], "kernel_ms_ncu": t_s * 1e3, "sm_clock_mhz": clk / 1e6,
        "warp_instructions": inst, "warp_rounds": rounds, "warp_instructions_per_round": inst / rounds,
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "time_at_full_issue_ms": t_full * 1e3, "issue_roofline_frac": t_full / t_s,
        "top_stalls_per_issue": top,
        "registers_per_thread": num(d, "launch__registers_per_thread"),
        "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "dram_bytes_per_launch": dram,
        "l2_sectors_per_launch": num(d, "lts__t_sectors.sum"),
        "l2_hit_rate_pct": num(d, "lts__t_sector_hit_rate.pct"),
        "source": rep.split("/")[-1],
    }
    for pipe in ("alu", "fma", "xu", "tex", "fp64"):
        k = f"sm__inst_executed_pipe_{pipe}.avg.pct_of_peak_sustained_active"
        if k in d:
            out[f"pipe_{pipe}_pct"] = num(d, k)
    if "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed" in d:
        out["pipe_fmaheavy_cycles_pct"] = num(d, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+", help="stream@N@B=path.ncu-rep")
    a = ap.parse_args()
    res = {"how": "ncu --set full --clock-control none over scripts/prof_step.py; scripts/issue_block.py"}
    for spec in a.reports:
        key, rep = spec.split("=", 1)
        name, n, b = key.split("@")
        res[f"{name}@{n}"] = dict(block(rep, int(n), int(b)), n=int(n), b=int(b))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

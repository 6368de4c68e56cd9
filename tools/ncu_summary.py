#!/usr/bin/env python
"""Summarise an ncu --set full report (per kernel) into profiles/<name>.md and
update profiles/traffic.json (dram bytes per launch of each hot kernel, read by
bench.py for the roofline "traffic" field).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_kernels.md
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "LSU wavefronts % (smem+L1)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
]

KEYS = {"k_median3_f32": "median", "k_gauss_tri<8": "gaussian", "k_median3_plane": "median_plane", "k_box_stream": "mean", "k_gauss_p2<8": "gaussian_p2", "k_gauss_ws<8": "gaussian_ws",
        "k_morph3": "erode", "k_log_stream": "log_stage2", "k_exact_z2<8": "exact_z",
        "k_exact_yx<8": "exact_yx"}


def main(rep, out_md):
    """rep: one report or several joined with ','"""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary of `{Path(rep).name}`", "",
             "Captured with `ncu --set full --clock-control none --import-source on` (one GPU).",
             "Absolute times are cold/serialised replays; compare shares, not absolutes.", ""]
    traffic_path = Path("profiles/traffic.json")
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        lines.append(f"## `{name[:160]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in idx:
                lines.append(f"| {label} | {r[idx[m]]} {units[idx[m]]} |")
        lines.append("")
        try:
            rd = float(r[idx["dram__bytes_read.sum"]])
            wr = float(r[idx["dram__bytes_write.sum"]])
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            rd *= scale.get(units[idx["dram__bytes_read.sum"]], 1.0)
            wr *= scale.get(units[idx["dram__bytes_write.sum"]], 1.0)
            for k, v in KEYS.items():
                if k in name:
                    traffic[v] = int(rd + wr)
        except (KeyError, ValueError):
            pass
    Path(out_md).write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print(f"wrote {out_md}; traffic {traffic}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

"""Summarise an `ncu --set full` capture of the step's stage kernels into
profiles/ (developer tool).

    python scripts/summarize_stage_ncu.py REPORT.ncu-rep OUT.txt "header line"

Prints, per captured launch, the metrics that decide these kernels' bound:
duration, issue activity, warps active, LSU pipe use, L1 / L2 hit rates,
DRAM bytes, registers and occupancy limit, instructions, top stall reasons."""
import csv
import io
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def main(rep, out, header):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    lines = [header, ""]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        lines.append(d.get("Kernel Name", "?").split("(")[0])
        for m in KEEP:
            if m in d:
                lines.append(f"  {m:<80} {d[m]} {u.get(m, '')}")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])

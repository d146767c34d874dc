"""Summarise one profiling round into profiles/ (developer tool).

    python scripts/summarize_profiles.py TAG

reads gpurun_out/bench_TAG.json, bench_ref_TAG.json, launches_TAG.csv and
k_pcg_TAG.ncu-rep (ncu --set full of the first timed bench step), writes
profiles/TAG_bench_c3.json, TAG_bench_ref_c3.json, TAG_launches_bench_c3.csv,
TAG_k_pcg_ncu_metrics.json and pcg_dram_bytes.json, and prints a markdown
section for profiles/README.md.
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
N, NU = 4194304, 3999992
KEEP = ("gpu__time_duration.sum", "dram__bytes", "dram__throughput", "sm__inst_executed.sum.pct",
        "smsp__issue_active", "sm__warps_active", "lts__t_sector_hit_rate", "launch__",
        "smsp__average_warps_issue_stalled", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(float)
    for r in rows[hi + 1:]:
        if len(r) > iv:
            try:
                agg[r[ik].split("(")[0].replace("void ", "").replace("cw::", "").replace("cwv::", "")] += \
                    float(r[iv].replace(",", ""))
            except ValueError:
                pass
    tot = sum(agg.values())
    return sorted(((k, 100 * v / tot) for k, v in agg.items()), key=lambda x: -x[1])


def ncu_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    keep = {}
    for k, u, v in zip(r[0], r[1], r[2]):
        if k.startswith(KEEP) and v != "":
            keep[k] = {"value": v, "unit": u}
    return keep


def main(tag):
    b = json.load(open(os.path.join(OUT, f"bench_{tag}.json")))
    ref = json.load(open(os.path.join(OUT, f"bench_ref_{tag}.json")))
    shutil.copy(os.path.join(OUT, f"bench_{tag}.json"), os.path.join(PROF, f"{tag}_bench_c3.json"))
    shutil.copy(os.path.join(OUT, f"bench_ref_{tag}.json"), os.path.join(PROF, f"{tag}_bench_ref_c3.json"))
    shutil.copy(os.path.join(OUT, f"launches_{tag}.csv"), os.path.join(PROF, f"{tag}_launches_bench_c3.csv"))
    shares = launch_shares(os.path.join(PROF, f"{tag}_launches_bench_c3.csv"))
    log = open(os.path.join(OUT, f"ncu_full_{tag}.log")).read()
    iters = int(re.search(r'"pcg_iterations": \[(\d+)', log).group(1))
    m = ncu_metrics(os.path.join(OUT, f"k_pcg_{tag}.ncu-rep"))
    json.dump({"source": f"ncu --set full --clock-control none, k_pcg (whole grid), first timed step of "
                         f"`python bench.py --steps 3 --warmup 3 --no-cpu --no-design` (C3, dt 0.2), {iters} iterations",
               "metrics": m}, open(os.path.join(PROF, f"{tag}_k_pcg_ncu_metrics.json"), "w"), indent=1)
    rd = float(m["dram__bytes_read.sum"]["value"]) * SCALE[m["dram__bytes_read.sum"]["unit"]]
    wr = float(m["dram__bytes_write.sum"]["value"]) * SCALE[m["dram__bytes_write.sum"]["unit"]]
    alg = 20 * N + 8 * NU + 44 * iters * NU
    json.dump({"source": f"profiles/{tag}_k_pcg_ncu_metrics.json", "iterations": iters,
               "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": alg,
               "traffic_over_algorithmic": (rd + wr) / alg,
               "dram_bytes_per_unknown_per_iteration": (rd + wr) / (iters * NU)},
              open(os.path.join(PROF, "pcg_dram_bytes.json"), "w"), indent=1)
    dur = float(m["gpu__time_duration.sum"]["value"])
    issue = float(m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", {}).get("value", "nan"))
    hit = float(m.get("lts__t_sector_hit_rate.pct", {}).get("value", "nan"))
    regs = m.get("launch__registers_per_thread", {}).get("value")
    rf = b["roofline"]
    pcg = [v for k, v in shares if "k_pcg" in k][0]
    top = ", ".join(f"{k} {v:.1f}%" for k, v in shares[:6])
    print(f"""## {tag} — bench line (C3, dt 0.2, {b['steps']} timed steps): `{tag}_bench_c3.json`

| quantity | value |
|---|---|
| device-resident throughput | **{b['value']:.3g} cell-steps/s** ({b['ms_per_step']:.2f} ms/step) |
| end to end (host state in/out every step, {b['e2e']['h2d_bytes_per_step'] / 1e6:.0f} MB each way) | {b['e2e']['value']:.3g} cell-steps/s |
| reference arm (`--impl reference`, oracle port, {ref['cpu_baseline']['cores']} host threads) | {ref['value']:.3g} cell-steps/s |
| CPU port, 1 core (bench `cpu_baseline`) | {b['cpu_baseline']['value']:.3g} cell-steps/s |
| k_pcg achieved algorithmic bandwidth | {rf['achieved']:.0f} GB/s = **{rf['frac']:.3f}** of the measured {rf['peak']:.0f} GB/s |
| k_pcg share of the step | {100 * rf['pcg_share_of_step']:.1f}% (events) / {pcg:.1f}% (ncu launch list) |
| seconds per design evaluation (C4 recipe, {b['design_eval']['settle_steps']} settle steps) | {b['design_eval']['seconds_per_evaluation']:.2f} s |
| clocks | {b['clocks']['sm_mhz']:.0f} MHz (max {b['clocks']['sm_max_mhz']:.0f}), {b['clocks']['samples']} samples, reasons {b['clocks']['reasons']} |

Launch list `{tag}_launches_bench_c3.csv`: {top}.

`k_pcg` capture `{tag}_k_pcg_ncu_metrics.json` (first timed step, {iters} iterations, {dur:.1f} ms
under ncu): DRAM {rd / 1e9:.1f} GB read + {wr / 1e9:.1f} GB write = {(rd + wr) / alg:.2f}x the
algorithmic bytes ({(rd + wr) / (iters * NU):.1f} B per unknown per iteration against 44); issue
active {issue:.1f}%, L2 hit rate {hit:.1f}%, {regs} registers.
""")


if __name__ == "__main__":
    main(sys.argv[1])

"""Per-kernel DRAM table of the last two bench steps (developer tool).

    python scripts/summarize_stepk.py TAG

reads gpurun_out/stepk_TAG.csv (ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum of `bench.py --steps 2 --warmup 3
--no-cpu --no-design`; the last two k_pcg launches and everything between
and after them are the e2e leg's two steps) and writes
profiles/TAG_step_kernels_dram.md."""
import collections
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = 6553.0


def main(tag):
    rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f"stepk_{tag}.csv"))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "").replace("cw::", "").replace("cwv::", "")
        d = launches.setdefault(int(r[iid]), {"name": name})
        d[r[im]] = float(r[iv].replace(",", ""))
    ids = list(launches)
    pcg = [i for i in ids if launches[i]["name"].startswith("k_pcg")]
    # the second-to-last step: from the k_report_init before its PCG launch,
    # plus the layout conversions of its uploads right before that
    start = ids.index(pcg[-2])
    while start > 0 and launches[ids[start]]["name"] != "k_report_init":
        start -= 1
    while start > 0 and launches[ids[start - 1]]["name"].startswith("k_ref_to_dev"):
        start -= 1
    stop = len(ids)
    for q in range(ids.index(pcg[-1]) + 1, len(ids)):   # the last step ends with its report commit
        if launches[ids[q]]["name"] == "k_report_commit":
            stop = q + 1
            break
    ids = ids[:stop]
    agg = collections.OrderedDict()
    for i in ids[start:]:
        L = launches[i]
        a = agg.setdefault(L["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += L.get("gpu__time_duration.sum", 0.0)
        a[2] += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
    out = [f"Per-kernel DRAM traffic over the last 2 C3 steps of `bench.py --steps 2 --warmup 3 --no-cpu "
           f"--no-design` (ncu, cold-cache, serialised; the e2e leg's steps, so the layout kernels appear, and "
           f"its first step builds the boundary lists of the reference-layout state's labels: k_bc_*_list, "
           f"k_bc_compose_*, the cub sort run once per labels array), "
           f"peak = measured copy bandwidth {PEAK:.0f} GB/s", "",
           "| kernel | launches/step | us/launch | DRAM MB/launch | DRAM GB/s | frac of peak |", "|---|---|---|---|---|---|"]
    for name, (n, ns, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        us = ns / n / 1e3
        mb = by / n / 1e6
        gbs = by / ns if ns else 0.0
        out.append(f"| {name} | {n / 2:.1f} | {us:.1f} | {mb:.1f} | {gbs:.0f} | {gbs / PEAK:.2f} |")
    path = os.path.join(ROOT, "profiles", f"{tag}_step_kernels_dram.md")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])

"""Per-kernel DRAM evidence for one C3 step (developer tool).

    python scripts/summarize_step_kernels.py IN.csv OUT.md STEPS

IN.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --csv` over `bench.py --steps STEPS --warmup 3 --no-cpu --no-design`.
Only the launches of the last STEPS steps are kept (from the predictor launch before the
first of the last STEPS k_pcg launches).  Per kernel: mean duration, DRAM bytes, achieved DRAM GB/s and the
fraction of the measured copy bandwidth (MEASURED_PEAKS.json), next to the algorithmic bytes
per launch where SURVEY.md 8d defines them.  ncu times are cold-cache and serialised.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 4194304                      # C3 cells
ALGO = {                         # algorithmic bytes per launch
    "k_mac_predict": 40 * N,     # u,v,w,k,omega in; u~,v~,w~,k',omega' out
    "k_mac_correct": 36 * N,     # u,v,w,u~,v~,w~ in; u',v',w' out
    "k_speed_max_flat": 12 * N,  # u,v,w in
    "k_div_max": 13 * N,         # u,v,w,labels in
    "k_cell_speed": 16 * N,      # u,v,w in; speed out
    "k_diffuse": 28 * N,         # u,v,w,nu_t in; u,v,w out
    "k_drag": 32 * N,            # u,v,w,g,speed in; u,v,w out
    "k_gradient": 29 * N,        # u,v,w,p,labels in; u,v,w out
    "k_turbulence": 36 * N,      # u,v,w,k,omega,nu_t in; k,omega,nu_t out
}
# k_pcg: 20 N + 8 Nu + 44 I Nu per launch with I that launch's iterations (bench.py roofline)


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    iid, ik, im, iu, iv = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "").replace("cw::", "").replace("cwv::", "")
        name = name.split("<")[0]
        d = launches.setdefault(int(r[iid]), {"name": name})
        d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    return list(launches.values())


def main(src, dst, steps):
    ls = load(src)
    last_vox = max([i for i, l in enumerate(ls) if l["name"].startswith("k_vox")] or [-1])
    ls = ls[last_vox + 1:]
    # the last STEPS steps: from the predictor before the first of the last STEPS k_pcg launches
    pcg = [i for i, l in enumerate(ls) if l["name"] == "k_pcg"]
    first = pcg[-steps] if len(pcg) >= steps else 0
    pred = [i for i, l in enumerate(ls[:first]) if l["name"] == "k_mac_predict"]
    ls = ls[pred[-1] if pred else first:]
    agg = collections.OrderedDict()
    for l in ls:
        a = agg.setdefault(l["name"], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += l.get("gpu__time_duration.sum", 0.0)
        a[2] += l.get("dram__bytes_read.sum", 0.0)
        a[3] += l.get("dram__bytes_write.sum", 0.0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.3)
    out = [f"Per-kernel DRAM traffic over {steps} C3 steps (ncu, cold-cache, serialised), "
           f"peak = measured copy bandwidth {peak:.0f} GB/s\n",
           "| kernel | launches/step | us/launch | DRAM MB/launch | DRAM GB/s | frac of peak | algorithmic MB/launch | algorithmic GB/s |",
           "|---|---|---|---|---|---|---|---|"]
    tot = sum(a[1] for a in agg.values())
    for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        us = 1e6 * t / n
        mb = (rd + wr) / n / 1e6
        gbs = (rd + wr) / t / 1e9 if t else 0.0
        al = ALGO.get(name)
        out.append(f"| {name} | {n / steps:.1f} | {us:.1f} | {mb:.1f} | {gbs:.0f} | {gbs / peak:.2f} | "
                   f"{al / 1e6 if al else float('nan'):.1f} | {(al * n / t / 1e9) if al else float('nan'):.0f} |")
    out.append(f"\nTotal {1e3 * tot / steps:.3f} ms per step under ncu.")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 2)

"""SURVEY §8(d)'s three views of the SA and LCP kernels on C3 (the 1M
window): from an ncu metrics CSV of one C3 analysis (bench.py --config C3),
per kernel class the summed time, DRAM bytes (view 1), L2 bytes (view 2) and
the modelled algorithmic bytes (view 3), each as GB/s and as a fraction of
the measured HBM peak.
    python tools/c3_views.py ncu.csv STEPS"""
import csv
import collections
import json
import os
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v *= {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(u, 1e-9)
    else:
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    per[r[ii]]["name"] = r[ki]
    per[r[ii]][r[mi]] = v
N = 1 << 20
# modelled (algorithmic) bytes per launch: K1 digit pass reads
# and writes each (u64 key, u32 value) once; the Manber-Myers key build reads
# SA + two ranks and writes key + value; the rank scan reads the sorted key
# and value and scatters the rank; PLCP: tokens at i and phi[i] + phi + PLCP
model = {"k_onesweep": 24 * N, "k_mm_keys": 24 * N, "k_double_keys": 20 * N, "k_scan<1, apo::{anonymous}::DoubleRankF>": 20 * N,
         "k_plcp": 16 * N, "k_phi": 12 * N}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for k, d in per.items():
    nm = d["name"]
    m = re.match(r"(?:void )?(?:apo::)?(?:\(anonymous namespace\)::|<unnamed>::)?([\w:]+(?:<[^(]*>)?)", nm)
    key = m.group(1) if m else nm[:40]
    base = key.split("<")[0]
    if base not in ("k_onesweep", "k_mm_keys", "k_double_keys", "k_plcp", "k_phi", "k_pos_of_zero") and "DoubleRankF" not in key:
        continue
    cls = "k_scan<DoubleRankF>" if "DoubleRankF" in key else base
    a = agg[cls]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    a[3] += d.get("lts__t_bytes.sum", 0)
    a[4] += {"k_onesweep": 24, "k_mm_keys": 24, "k_double_keys": 20, "k_scan<DoubleRankF>": 20, "k_plcp": 16,
             "k_phi": 12}.get(cls, 0) * N
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6547.2) if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6547.2
out = {}
print(f"{'kernel':24s} {'launches/step':>13s} {'ms/step':>8s} {'DRAM GB/s':>10s} {'L2 GB/s':>9s} {'model GB/s':>11s}  fractions of {peak:.0f} GB/s (DRAM / L2 / model)")
for cls, (n, t, dr, l2, mo) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    v1, v2, v3 = dr / t / 1e9, l2 / t / 1e9, mo / t / 1e9
    out[cls] = {"launches_per_step": n / steps, "ms_per_step": 1e3 * t / steps, "dram_gbs": v1, "l2_gbs": v2, "model_gbs": v3,
                "frac_dram": v1 / peak, "frac_l2": v2 / peak, "frac_model": v3 / peak}
    print(f"{cls:24s} {n / steps:13.1f} {1e3 * t / steps:8.3f} {v1:10.0f} {v2:9.0f} {v3:11.0f}  "
          f"{v1 / peak:.3f} / {v2 / peak:.3f} / {v3 / peak:.3f}")
json.dump({"peak_gbs": peak, "n": N, "kernels": out}, open(sys.argv[1] + ".views.json", "w"), indent=1)

"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
five step kernels from an ncu --set full raw page (csv or csv.gz), merged into
profiles/ncu_traffic.json[workload][f32|f64] (what bench.py reports as
roofline.traffic):  python tools/ncu_traffic.py raw.csv.gz film512 f32 "source note"
"""
import csv
import gzip
import json
import os
import sys

path, workload, prec, note = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else ""
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
h, units = rows[0], rows[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
names = {"k_r2c_x": "k_r2c_x", "k_fft_y_fwd": "k_fft_y_fwd", "k_fft_z_conv": "k_fft_z_conv",
         "k_fft_y_inv": "k_fft_y_inv", "k_c2r_x_llg": "k_c2r_x_llg"}
out = {}
for r in rows[2:]:
    if len(r) <= max(ir, iw):
        continue
    kname = r[ik]
    key = next((v for k, v in names.items() if k in kname.split("<")[0]), None)
    if key is None:
        continue
    b = float(r[ir]) * UNIT[units[ir]] + float(r[iw]) * UNIT[units[iw]]
    out.setdefault(key, []).append(b)
res = {k: int(sum(v) / len(v)) for k, v in out.items()}
dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
try:
    d = json.load(open(dst))
except Exception:
    d = {}
if not isinstance(d.get(workload, {}).get(prec, None), (dict, type(None))) or (workload in d and "f32" not in d[workload] and "f64" not in d[workload]):
    d[workload] = {}   # old layout (keyed by workload only)
d.setdefault(workload, {})[prec] = res
d.setdefault("_source", {})
if not isinstance(d["_source"], dict):
    d["_source"] = {}
d["_source"][f"{workload}/{prec}"] = note
json.dump(d, open(dst, "w"), indent=1, sort_keys=True)
print(workload, prec, res)

"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, unit
-aware) of the attempt kernels in an ncu --set full report, keyed by the
bench.py stage names; K1 = k_warp_moving + k_lncc_fwd.  Usage:
  python tools/ncu_traffic.py REPORT.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    return float(r[ix[name]].replace(",", "")) * SCALE.get(units[ix[name]], 1.0)


per = {}
for r in data:
    k = r[ix["Kernel Name"]]
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    t = float(r[ix["gpu__time_duration.sum"]].replace(",", "")) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "ms": 1e-3,
                                                                   "msecond": 1e-3}.get(units[ix["gpu__time_duration.sum"]], 1)
    per.setdefault(k.split("(")[0].replace("void ", "").split("<")[0], []).append((b, t))
stage = {"K1_lncc_fwd": ["k_warp_moving", "k_lncc_fwd"], "K2_lncc_bwd": ["k_lncc_bwd"],
         "K3_step_smooth": ["k_step_smooth"], "K4_compose_smooth": ["k_compose_smooth"]}
out = {}
for s, ks in stage.items():
    if all(k in per for k in ks):
        out[s] = sum(sum(b for b, _ in per[k]) / len(per[k]) for k in ks)
for k, v in per.items():
    print(f"{k:20s} launches {len(v)}  DRAM bytes/launch {sum(b for b, _ in v) / len(v):.4g}  "
          f"time/launch {sum(t for _, t in v) / len(v) * 1e3:.4f} ms")
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)

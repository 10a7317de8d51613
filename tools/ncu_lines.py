"""Per-CUDA-source-line instruction and stall totals of one kernel in an ncu
report (needs -lineinfo and --import-source on).  Usage:
  python tools/ncu_lines.py REPORT.ncu-rep [top_n] [--smem] [--kernel REGEX]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
kfilter = []
if "--kernel" in sys.argv:
    kfilter = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]]
out = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
fname = None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "Function Name" or len(row) < len(hdr):
        continue
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    wf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
    wx = hdr.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in hdr else None
    try:
        line = int(row[0])
    except ValueError:
        continue
    # rows carry the CUDA line in col 0/1 and a SASS instruction in col 3
    key = (fname, line, row[1].strip()[:90])
    a = agg.setdefault(key, [0.0, 0.0, 0.0, 0.0])
    def num(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    a[0] += num(row[ie])
    a[1] += num(row[st])
    if wf is not None:
        a[2] += num(row[wf])
        a[3] += num(row[wx])
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
tot_w = sum(v[2] for v in agg.values()) or 1
key = 2 if "--smem" in sys.argv else 0
print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}, shared wavefronts {tot_w:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{100 * v[0] / tot_i:6.2f}% inst {100 * v[1] / tot_s:6.2f}% stall {100 * v[2] / tot_w:6.2f}% smem-wf "
          f"(excess {v[3]:.2e})  {k[0]}:{k[1]}  {k[2]}")

"""Summarise an ncu --set full report: key throughput / stall metrics per kernel,
and the SASS opcode mix of one kernel.  Usage:
  python tools/ncu_summary.py REPORT.ncu-rep [kernel-regex-for-opcode-mix]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "local_load_bytes" if "local_load_bytes" in idx else "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum"]
stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
print("kernel".ljust(58), " | ".join(r[idx["Kernel Name"]][:18] for r in data))
for w in want:
    if w in idx:
        print(w[:58].ljust(58), " | ".join(r[idx[w]][:18] for r in data))
tot = [sum(float(r[idx[s]] or 0) for s in stalls) or 1 for r in data]
top = sorted(stalls, key=lambda s: -sum(float(r[idx[s]] or 0) for r in data))[:8]
for s in top:
    print(("stall " + s.replace("smsp__pcsamp_warps_issue_stalled_", ""))[:58].ljust(58),
          " | ".join(f"{float(r[idx[s]] or 0) / t * 100:5.1f}%" for r, t in zip(data, tot)))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + sys.argv[2]],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    d = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
    ia, ie, isamp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ops, st, tot = collections.Counter(), collections.Counter(), 0
    for r in d:
        toks = r[ia].split()
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ops[op] += float(r[ie] or 0); st[op] += float(r[isamp] or 0); tot += float(r[ie] or 0)
    print(f"opcode mix of {sys.argv[2]} ({tot:.3g} warp instrs):")
    for op, v in ops.most_common(16):
        print(f"  {op:10s} {v / tot * 100:5.1f}%  stall-samples {st[op]:.0f}")

"""Static SASS summary of the hot kernels in the built library (no GPU):
registers, spills and the counts of the instructions that identify the
design (UTMALDG = TMA tensor loads, LDGSTS = cp.async, DFMA/DADD/DMUL = fp64,
F2F = fp32<->fp64 conversions, LDS/STS shared, LDG/STG global, BAR, SHFL).
    python tools/sass_summary.py [lib] > profiles/r02/sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2603_19371_b200", "libwarplm_b200.so")
KERNELS = {
    "K1a k_warp_moving<true>": r"_ZN3wlm13k_warp_movingILb1EEEvNS_5BatchEiii",
    "K1b k_lncc_fwd<2>": r"_ZN3wlm10k_lncc_fwdILi2EEEvNS_5BatchEi",
    "K2 k_lncc_bwd<2,false>": r"_ZN3wlm10k_lncc_bwdILi2ELb0EEEvNS_5BatchENS_8LmParamsEi",
    "K2 k_lncc_bwd<2,true> (low memory)": r"_ZN3wlm10k_lncc_bwdILi2ELb1EEEvNS_5BatchENS_8LmParamsEi",
    "K3 k_step_smooth<3,false>": r"_ZN3wlm13k_step_smoothILi3ELb0EEEvNS_5BatchENS_8LmParamsEi",
    "K4 k_compose_smooth<2,true> (TMA)": r"_ZN3wlm16k_compose_smoothILi2ELb1EEEvNS_5BatchENS_8LmParamsEi14CUtensorMap_st",
}
OPS = ["UTMALDG", "LDGSTS", "DFMA", "DADD", "DMUL", "F2F", "LDS", "STS", "LDG", "STG", "BAR", "SHFL", "MUFU"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
print(f"library: {os.path.relpath(lib, ROOT)}  (cuobjdump -sass / -res-usage, static counts)")
print("kernel".ljust(38) + "regs  " + " ".join(o.rjust(7) for o in OPS))
for name, mangled in KERNELS.items():
    body = next((f for f in funcs if f.startswith(mangled)), None)
    if body is None:
        print(name.ljust(38) + "  (not found)")
        continue
    cnt = collections.Counter()
    for line in body.splitlines():
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            cnt[m.group(1).split(".")[0]] += 1
    r = re.search(re.escape(mangled) + r"[^\n]*\n\s*REG:(\d+)", res)
    regs = r.group(1) if r else "?"
    print(name.ljust(38) + regs.rjust(4) + "  " + " ".join(str(cnt[o]).rjust(7) for o in OPS))

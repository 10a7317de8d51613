#!/bin/bash
# A/B the default library against build/var_*/ variants on the default bench
# (per-kernel CUDA-event times), alternating twice.
#   gpurun --timeout 900 -- 'bash tools/ab_bench.sh k2s8 k2s2'
set -u
mkdir -p gpurun_out
run() {
  local tag=$1 lib=$2
  WLM_LIB_PATH=$lib python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline --e2e-iters 1 --pairs-per-gpu ${PAIRS:-8} \
    > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{t}.json"))
    print(f"{t:10s} {d['value']:8.4f} Gvox/s", {k: v for k, v in d["roofline"]["per_kernel_ms"].items()})
except Exception as e:
    print(t, "failed", e)
PY
}
for rep in 1 2; do
  [ "${SKIPBASE:-0}" = 1 ] || run base ""
  for v in "$@"; do run $v build/var_$v/libwarplm_b200.so; done
done

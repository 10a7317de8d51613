#!/bin/bash
# A/B the default library under environment settings (tag=VAR=val,VAR=val):
#   gpurun -- 'bash tools/ab_env.sh rows2=WLM_K1A_ROWS=2 prio=WLM_K1A_PRIO=1'
set -u
mkdir -p gpurun_out
run() {
  local tag=$1 envs=$2
  env ${envs//,/ } python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline --e2e-iters 1 \
    --pairs-per-gpu ${PAIRS:-64} > gpurun_out/abe_$tag.json 2> gpurun_out/abe_$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/abe_{t}.json"))
    print(f"{t:10s} {d['value']:8.4f} Gvox/s {d['ms_per_step']:.3f} ms", {k: v for k, v in d["roofline"]["per_kernel_ms"].items()})
except Exception as e:
    print(t, "failed", e)
PY
}
for rep in 1 2; do
  run base "WLM_AB_BASE=1"
  for v in "$@"; do run ${v%%=*} "${v#*=}"; done
done

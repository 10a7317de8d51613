#!/bin/bash
# Pair-group count A/B on the default config-4 batch (64 pairs per GPU).
set -u
mkdir -p gpurun_out
for rep in 1 2; do
  for g in 1 2 3 4; do
    WLM_PAIR_GROUPS=$g python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline --e2e-iters 1 \
      > gpurun_out/grp_$g.json 2> gpurun_out/grp_$g.err
    python -c "import json;d=json.load(open('gpurun_out/grp_$g.json'));print('groups $g', d['value'], d['ms_per_step'])"
  done
done

#!/bin/bash
# One gpurun call: the default bench line, the ncu launch list of a short
# bench, and one ncu --set full capture of the attempt kernels (each ncu run
# only after the same command exited 0 without ncu).
#   gpurun --timeout 1500 -- 'bash tools/profile_round.sh'
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
SHORT="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-iters 1"
$SHORT > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 49 --csv \
      --log-file gpurun_out/launches_final.csv $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
# the full capture profiles whole-batch launches (one pair group), the unit
# bench.py's per-stage CUDA-event times and roofline.traffic refer to
$SHORT > gpurun_out/plain2.log 2>&1 && WLM_PAIR_GROUPS=1 \
  ncu --set full --clock-control none --import-source on \
      -k regex:'k_warp_moving|k_lncc_fwd|k_plane_sums|k_finalize|k_lncc_bwd|k_step_smooth|k_compose_smooth' -s 14 -c 7 \
      -o gpurun_out/prof_final $SHORT > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"

#!/bin/bash
# Round-2 measurement call (one gpurun):
#   gpurun --timeout 3000 -- 'bash tools/profile_r02.sh'
# 1. the default bench line (config 4, 64 pairs) with cpu_baseline + CPU tables
# 2. ncu launch list of a short run of the same command (--clock-control none)
# 3. one ncu --set full capture of the attempt kernels on whole-batch launches
#    (WLM_PAIR_GROUPS=1), each only after the same command exited 0 without ncu
# 4. config 5 at 1024^3 (one slab group on one GPU)
# 5. the reference arm (CPU)
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > gpurun_out/r02_gpu.txt
python bench.py --cpu-tables --table6 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
SHORT="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --e2e-iters 1"
$SHORT > gpurun_out/r02_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv \
      --log-file gpurun_out/r02_launches.csv $SHORT > gpurun_out/r02_ncu_launch.log 2>&1; echo "launches rc=$?"
$SHORT > gpurun_out/r02_plain2.log 2>&1 && WLM_PAIR_GROUPS=1 \
  ncu --set full --clock-control none --import-source on \
      -k regex:'k_warp_moving|k_lncc_fwd|k_plane_sums|k_finalize|k_lncc_bwd|k_step_smooth|k_compose_smooth' -s 14 -c 7 \
      -o gpurun_out/r02_prof $SHORT > gpurun_out/r02_ncu_full.log 2>&1; echo "full rc=$?"
python bench.py --config 5 --steps 5 --warmup 3 --e2e-iters 5 > gpurun_out/r02_config5.json 2> gpurun_out/r02_config5.err; echo "config5 rc=$?"
python bench.py --impl reference > gpurun_out/r02_reference.json 2> gpurun_out/r02_reference.err; echo "reference rc=$?"

set -u
mkdir -p gpurun_out
SHORT="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra --e2e-iters 1 --pairs-per-gpu 8"
$SHORT > gpurun_out/plain.log 2>&1; echo plain rc=$?
WLM_PAIR_GROUPS=1 ncu --set full --clock-control none --import-source on \
  -k regex:'k_lncc_fwd|k_lncc_bwd|k_step_smooth|k_compose_smooth|k_warp_moving' -s 10 -c 5 \
  -o gpurun_out/prof_r2a $SHORT > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
ls -la gpurun_out

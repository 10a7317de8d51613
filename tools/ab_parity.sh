#!/bin/bash
# A/B one variant against the default and run a parity subset on it:
#   gpurun -- 'bash tools/ab_parity.sh VARIANT'
v=$1
bash tools/ab_bench.sh $v 2>&1 | grep Gvox
WLM_LIB_PATH=build/var_$v/libwarplm_b200.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu \
  -k "config1 or degenerate or random_configs_match or pair_groups or slab_group_is" 2>&1 | tail -2

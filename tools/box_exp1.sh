#!/bin/bash
# GEMM K3 variants (C2 per level) and the tile memory cap at C3.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py -q > gpurun_out/e1_configs.log 2>&1
python tools/level_times.py C2 dmma > gpurun_out/e1_lt_ks2rb2.log 2>&1
for v in ks1 rb3 ks3 rb1ks4; do
  IFGF_B200_LIB=$PWD/paper_2112_15198_b200/libifgf_b200_$v.so python tools/level_times.py C2 dmma > gpurun_out/e1_lt_$v.log 2>&1
done
python tools/level_times.py C3 > gpurun_out/e1_lt_c3_cap8.log 2>&1
IFGF_TILE_MAX_GB=40 python tools/level_times.py C3 > gpurun_out/e1_lt_c3_cap40.log 2>&1

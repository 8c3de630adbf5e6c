#!/bin/bash
# Tile memory cap: full applies (setup + passes) of C3, C4, C5 at 8 and 32 GB.
mkdir -p gpurun_out
IFGF_TILE_MAX_GB=8 python tools/config_run.py C3 C4 C5 > gpurun_out/e2_cap8.log 2>&1
IFGF_TILE_MAX_GB=32 python tools/config_run.py C3 C4 C5 > gpurun_out/e2_cap32.log 2>&1
nvidia-smi --query-gpu=memory.total --format=csv >> gpurun_out/e2_cap32.log

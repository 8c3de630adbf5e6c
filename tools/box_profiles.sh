#!/bin/bash
# ncu evidence for the round's bench (logs and reports to gpurun_out/).
mkdir -p gpurun_out
# 1. launch list of the bench command (cold, serialised per-launch times: compare shares)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-e2e \
  --no-cpu-baseline > gpurun_out/launches_r02.log 2>&1
# 2. DRAM bytes of every K1-K4 launch of one C2 apply (bench.py roofline.traffic)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"k_(near|level_d|propagate|interp)" --csv \
  --log-file gpurun_out/dram_r02.csv python tools/profile_step.py C2 1 > gpurun_out/dram_r02.log 2>&1
# 3. full sets of the largest K3 (d=7 rows launch) and a K4 launch
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_propagate_rows \
  --launch-skip 1 -c 1 -o gpurun_out/ncu_r02_k3 python tools/profile_step.py C2 1 > gpurun_out/ncu_r02_k3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_interp \
  --launch-skip 2 -c 1 -o gpurun_out/ncu_r02_k4 python tools/profile_step.py C2 1 > gpurun_out/ncu_r02_k4.log 2>&1
echo done > gpurun_out/profiles_done

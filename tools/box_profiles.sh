#!/bin/bash
# ncu evidence for the round's bench (logs and reports to gpurun_out/).
mkdir -p gpurun_out
# 0. tests, per-level K3 times, microbenchmarks
python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_all.log
{ echo "# tools/level_times.py C2 rows"; python tools/level_times.py C2 rows | tail -6;
  echo "# tools/level_times.py C2 dmma (warp GEMM on every tiled level)"; python tools/level_times.py C2 dmma | tail -6;
  echo "# tools/level_times.py C2 auto (default)"; IFGF_G4_TRACE=1 python tools/level_times.py C2 auto 2>&1 | tail -9;
  echo "# tools/prop_modes.py C2 / C1"; python tools/prop_modes.py C2 node rows fly dmma auto; python tools/prop_modes.py C1 rows dmma auto; } > gpurun_out/levels_rows_vs_wgemm.log 2>&1
{ echo "# tools/micro/ldg_share"; tools/micro/ldg_share; echo "# tools/micro/lds_bcast"; tools/micro/lds_bcast; } > gpurun_out/micro_block_loads.log 2>&1
python tools/config_work.py C2 C3 C4 C5 > gpurun_out/config_work_c2_c5.log 2>&1
# 1. bench (default run) and the multi-GPU entry at world 1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
# 2. launch list of the bench command (cold, serialised per-launch times: compare shares)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv \
  --log-file gpurun_out/launches_c2_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e \
  --no-cpu-baseline > gpurun_out/launches_c2_bench.log 2>&1
# 3. DRAM bytes of every K1-K4 launch of one C2 apply (bench.py roofline.traffic)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"k_(near|level_d|propagate|interp)" --csv \
  --log-file gpurun_out/dram_c2_all_launches.csv python tools/profile_step.py C2 1 > gpurun_out/dram_c2.log 2>&1
# 4. full sets: the warp GEMM (d = 8, 7, 6 launches), the rows kernel (d = 5), K4
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_propagate_wgemm \
  -c 3 -f -o gpurun_out/ncu_c2_k3_wgemm python tools/profile_step.py C2 1 > gpurun_out/ncu_c2_k3_wgemm.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_propagate_rows \
  -c 1 -f -o gpurun_out/ncu_c2_k3_rows python tools/profile_step.py C2 1 > gpurun_out/ncu_c2_k3_rows.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_interp \
  --launch-skip 2 -c 1 -f -o gpurun_out/ncu_c2_k4 python tools/profile_step.py C2 1 > gpurun_out/ncu_c2_k4.log 2>&1
# 5. the setup's locate kernel (K4 records), two of its six launches
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_locate_points \
  --launch-skip 6 -c 2 -f -o gpurun_out/ncu_c2_locate python tools/profile_step.py C2 1 --setups 2 > gpurun_out/ncu_c2_locate.log 2>&1
# 6. K4 from the records against the locate-per-pair K4 (bitwise, per-level times)
python tools/k4_records.py C2 > gpurun_out/k4_records_c2.log 2>&1
# 7. summaries here (the reports themselves exceed what gpurun_out/ brings back)
for tag in ncu_c2_k3_wgemm ncu_c2_k3_rows ncu_c2_k4 ncu_c2_locate; do
  python tools/ncu_summary.py gpurun_out/$tag.ncu-rep gpurun_out/$tag > /dev/null 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv > gpurun_out/$tag.src.csv 2> /dev/null
  python tools/ncu_stalls.py gpurun_out/$tag.src.csv > gpurun_out/${tag}_stalls.txt 2>&1
  rm -f gpurun_out/$tag.src.csv gpurun_out/$tag.ncu-rep
done
echo done > gpurun_out/profiles_done

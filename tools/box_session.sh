#!/bin/bash
# One GPU-box session of checks and measurements (logs to gpurun_out/).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/s_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/s_gputests.log
timeout 600 python bench.py --steps 10 --warmup 5 > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/s_bench_ref.json 2> gpurun_out/s_bench_ref.err
timeout 300 python tools/e2e_probe.py C2 8 > gpurun_out/s_e2e.log 2>&1
timeout 300 python bench.py --dist --steps 5 --warmup 3 > gpurun_out/s_bench_dist.json 2> gpurun_out/s_bench_dist.err
IFGF_DIST_RANK_TIMING=1 timeout 600 python tools/partition_probe.py C4 8 > gpurun_out/s_partition_c4.log 2>&1
echo done > gpurun_out/s_done

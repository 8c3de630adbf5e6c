#!/bin/bash
# Round-end box run: GPU tests, smoke, default bench, then the full-size C3
# reference fixture (tests/golden/make_config_golden.py, ~1 h on the box's
# host cores) copied into gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/re_gpu_tests.log 2>&1; echo "TESTS_EXIT $?" >> gpurun_out/re_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/re_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err
nproc > gpurun_out/re_nproc.txt
( time timeout 6000 python tests/golden/make_config_golden.py C3 ) > gpurun_out/re_golden_c3.log 2>&1
cp tests/golden/config_C3.npz gpurun_out/ 2>/dev/null
echo DONE >> gpurun_out/re_golden_c3.log

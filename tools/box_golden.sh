#!/bin/bash
# Full-size parity fixture of C3 from the unmodified reference on the GPU box's
# host (16 cores, ~196 GB; the reference needs more memory than the 62 GB of
# the build container at C3).  Output to gpurun_out/.
mkdir -p gpurun_out
( free -g; nproc ) > gpurun_out/golden_box_host.txt
( time timeout 3300 python tests/golden/make_config_golden.py --checker reference \
    --threads 16 --out gpurun_out C3 ) > gpurun_out/golden_c3.log 2>&1
echo "C3 rc=$?" >> gpurun_out/golden_c3.log

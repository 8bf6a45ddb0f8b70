#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/fuse
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_gpu_parity.py -q -x -k "two_set or variants or c5_full or q1_rhs or q2_rhs" > gpurun_out/fuse/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/fuse/pytest.log
for t in fuse_sets=1 fuse_sets=0; do timeout 600 python tools/cfg_kernels.py C5 --tuning $t > gpurun_out/fuse/k_C5_$t.json 2>&1; echo $t=$?; done
timeout 600 python tools/kbench.py --reps 20 > gpurun_out/fuse/kbench.log 2>&1; tail -1 gpurun_out/fuse/kbench.log
timeout 600 python tools/kbench.py --reps 20 --tuning fuse_sets=0 > gpurun_out/fuse/kbench0.log 2>&1; tail -1 gpurun_out/fuse/kbench0.log

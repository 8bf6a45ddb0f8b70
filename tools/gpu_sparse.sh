#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sp
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/sp/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/sp/pytest.log
for t in sparse_warps=1 sparse_warps=2; do timeout 600 python tools/cfg_kernels.py C3 --reps 10 --tuning $t > gpurun_out/sp/k_C3_$t.json 2>&1; echo $t=$?; done
timeout 600 python tools/cfg_kernels.py C1 --reps 10 > gpurun_out/sp/k_C1.json 2>&1; echo C1=$?

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests/test_gpu_properties.py -q -x -k "q1_rhs or c5_full" > gpurun_out/q1/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/q1/pytest.log
timeout 600 python tools/cfg_kernels.py C5 > gpurun_out/q1/k_C5.json 2>&1; echo C5=$?

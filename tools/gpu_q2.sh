#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/q2
timeout 900 python -m pytest tests/test_gpu_properties.py -q -x -k "q1_rhs or q2_rhs or c5_full or dense_2d or q2_many" > gpurun_out/q2/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/q2/pytest.log
timeout 600 python tools/cfg_kernels.py C5 > gpurun_out/q2/k_C5.json 2>&1; echo C5=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5 or c2" > gpurun_out/q2/full.log 2>&1; echo full=$?; tail -3 gpurun_out/q2/full.log

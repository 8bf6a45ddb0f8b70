#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2b
timeout 600 env AK_LIB_PATH=$PWD/paper_2404_17344_b200/libaddkern_b200_checked.so python tools/sanitize_cases.py > gpurun_out/r2b/checked.log 2>&1; echo checked=$?; tail -3 gpurun_out/r2b/checked.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2b/pytest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r2b/pytest.log
timeout 600 python tools/cfg_kernels.py C5 > gpurun_out/r2b/k_C5.json 2>&1; echo C5=$?

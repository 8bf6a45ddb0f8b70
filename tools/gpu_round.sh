#!/bin/bash
# final round measurement (tools/gpu_final.sh) + the GPU suite on the product and on the checked library
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r2} bash tools/gpu_final.sh
mkdir -p gpurun_out/t
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t/pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/t/pytest.log
AK_LIB_PATH=$PWD/paper_2404_17344_b200/libaddkern_b200_checked.so timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t/pytest_checked.log 2>&1; echo checked=$?; tail -2 gpurun_out/t/pytest_checked.log

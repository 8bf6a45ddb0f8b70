#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_solver.py -m gpu -q -x -s -k "fullsize or c2_full or paper_bound or full" > gpurun_out/newtests.log 2>&1; echo newtests=$?
tail -30 gpurun_out/newtests.log

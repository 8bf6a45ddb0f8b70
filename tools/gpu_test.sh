#!/bin/bash
# the GPU test suite + per-kernel times of configs 3, 4 (kbench) and 5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/t
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t/pytest.log 2>&1; echo pytest=$?; tail -4 gpurun_out/t/pytest.log
timeout 600 python tools/kbench.py --reps 20 2>&1 | tail -1
for c in C5 C3; do timeout 600 python tools/cfg_kernels.py $c > gpurun_out/t/k_$c.json 2>&1; echo $c=$?; done

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2a
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2a/cases.log 2>&1; echo cases=$?; tail -2 gpurun_out/r2a/cases.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r2a/pytest.log
for c in C5 C3 C2; do timeout 600 python tools/cfg_kernels.py $c > gpurun_out/r2a/k_$c.json 2>&1; echo $c=$?; done
timeout 600 python tools/kbench.py --reps 20 > gpurun_out/r2a/kbench.log 2>&1; tail -1 gpurun_out/r2a/kbench.log

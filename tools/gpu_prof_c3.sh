#!/bin/bash
# C3 sparse q = 3 kernels: timing, then ncu --set full with source counters
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pc3
timeout 600 python tools/cfg_kernels.py C3 --reps 5 > gpurun_out/pc3/k_C3.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spread3w|k_interp3m" -s 0 -c 3 \
   -o gpurun_out/pc3/c3 python tools/cfg_kernels.py C3 --reps 1 > gpurun_out/pc3/ncu.log 2>&1; echo ncu=$?
tail -2 gpurun_out/pc3/ncu.log

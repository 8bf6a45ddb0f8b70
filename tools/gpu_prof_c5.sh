#!/bin/bash
# config 5: per-kernel timing, then one ncu --set full capture of every kernel family of a step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pc5
timeout 600 python tools/cfg_kernels.py C5 --reps 1 > gpurun_out/pc5/k_C5.json 2>&1 && \
timeout 2000 ncu --set full --clock-control none --import-source on \
   -k regex:"k_interp2r|k_spread2r|k_interp1r|k_spread1r|k_spread3r|k_interp3c" -s 0 -c 9 \
   -o gpurun_out/pc5/prof python tools/cfg_kernels.py C5 --reps 1 > gpurun_out/pc5/ncu.log 2>&1; echo ncu=$?
tail -2 gpurun_out/pc5/ncu.log

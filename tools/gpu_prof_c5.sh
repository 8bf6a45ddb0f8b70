#!/bin/bash
# C5 q<=2 kernels: parity, timing, then one ncu --set full capture of each
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pc5
timeout 900 python -m pytest tests/test_gpu_properties.py -q -x -k "q1_rhs" > gpurun_out/pc5/pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pc5/pytest.log
timeout 600 python tools/cfg_kernels.py C5 --reps 1 > gpurun_out/pc5/k_C5.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_interp2c|k_spread2c|k_interp1r|k_spread1r" -s 0 -c 6 \
   -o gpurun_out/pc5/prof python tools/cfg_kernels.py C5 --reps 1 > gpurun_out/pc5/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/pc5/ncu.log

#!/bin/bash
# q = 3 kernels: C4 (R = 1) spread/interp and C5 (R = 16) RHS-pair spread / interp, ncu --set full
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pq3
timeout 600 python bench.py --quick --steps 2 --warmup 1 > gpurun_out/pq3/plain4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spread3c|k_interp3c" -s 2 -c 2 \
   -o gpurun_out/pq3/c4 python bench.py --quick --steps 2 --warmup 1 > gpurun_out/pq3/ncu4.log 2>&1; echo ncu4=$?
timeout 600 python tools/cfg_kernels.py C5 --reps 1 > gpurun_out/pq3/plain5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spread3r|k_interp3c|k_interp2r|k_spread2r|k_interp1r|k_spread1r" -s 0 -c 7 \
   -o gpurun_out/pq3/c5 python tools/cfg_kernels.py C5 --reps 1 > gpurun_out/pq3/ncu5.log 2>&1; echo ncu5=$?
tail -2 gpurun_out/pq3/ncu5.log

#!/bin/bash
# ncu (--set full) of the sparse config-3 kernels for the main library and each tools/_var variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pv
timeout 900 ncu --set full --clock-control none -k regex:"${KREGEX:-k_interp3m}" -s 0 -c 1 \
   -o gpurun_out/pv/main python tools/cfg_kernels.py C3 --reps 1 > gpurun_out/pv/main.log 2>&1; echo main=$?
for f in tools/_var/*.so; do
  b=$(basename $f .so)
  AK_LIB_PATH=$PWD/$f timeout 900 ncu --set full --clock-control none -k regex:"${KREGEX:-k_interp3m}" -s 0 -c 1 \
     -o gpurun_out/pv/$b python tools/cfg_kernels.py C3 --reps 1 > gpurun_out/pv/$b.log 2>&1; echo $b=$?
done

#!/bin/bash
# ncu --set full (source counters) of one kernel family (KREGEX) in one step of config CFG
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pk
timeout 600 python tools/cfg_kernels.py ${CFG:-C3} --reps 3 > gpurun_out/pk/k.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-1} \
   -o gpurun_out/pk/${TAG:-prof} python tools/cfg_kernels.py ${CFG:-C3} --reps 1 > gpurun_out/pk/ncu.log 2>&1; echo ncu=$?
tail -2 gpurun_out/pk/ncu.log

#!/bin/bash
# round measurement: bench line (ours + reference arm), launch list of the same command,
# one full ncu capture of the dominant kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r2}
mkdir -p gpurun_out/$TAG
timeout 1500 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/$TAG/reference.json 2> gpurun_out/$TAG/reference.err; echo ref=$?
timeout 600 python bench.py --quick --steps 3 --warmup 3 > gpurun_out/$TAG/plain_quick.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/$TAG/launches.csv python bench.py --quick --steps 3 --warmup 3 > gpurun_out/$TAG/ncu_launches.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread3h|k_interp3c" -s 4 -c 2 \
   -o gpurun_out/$TAG/prof_full python bench.py --quick --steps 3 --warmup 3 > gpurun_out/$TAG/ncu_full.log 2>&1; echo full=$?

#!/bin/bash
# full bench line + reference arm (run under gpurun)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/bench
timeout 1200 python bench.py > gpurun_out/bench/ours.json 2> gpurun_out/bench/ours.err; echo ours=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench/ref.json 2> gpurun_out/bench/ref.err; echo ref=$?
timeout 120 python bench.py --gpus 2 > gpurun_out/bench/gpus2.out 2>&1; echo gpus2=$?
tail -c 600 gpurun_out/bench/ours.err

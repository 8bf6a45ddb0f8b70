#!/bin/bash
# quick loop: selected GPU tests (TESTS, pytest -k expression) + per-kernel times of configs 3, 4 and 5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/q
timeout 1500 python -m pytest tests -m gpu -q -x ${TESTS:+-k "$TESTS"} > gpurun_out/q/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/q/pytest.log
timeout 600 python tools/kbench.py --reps 20 2>&1 | tail -1
for c in ${CFGS:-C3 C5}; do timeout 600 python tools/cfg_kernels.py $c > gpurun_out/q/k_$c.json 2>&1; echo $c=$?; python -c "import json;d=json.load(open('gpurun_out/q/k_$c.json'));print('$c', round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"; done

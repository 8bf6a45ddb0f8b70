cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/q1
timeout 1200 python -m pytest tests -m gpu -q -x -k "q1 or fuzz or c5_full or families or variants or golden" > gpurun_out/q1/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/q1/pytest.log
CONFIG=C5 timeout 900 bash tools/gpu_var_cfg.sh

timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for s in 2 3 4; do AK_SUPERCELL3=$s timeout 300 python tools/kbench.py; done

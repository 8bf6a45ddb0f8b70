timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for s2 in 8 1; do AK_SUPERCELL2=$s2 timeout 600 python tools/cfg_time.py; done > gpurun_out/q2_time.log 2>&1
cat gpurun_out/q2_time.log

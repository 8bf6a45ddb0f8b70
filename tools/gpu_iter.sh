for i in 1 2; do timeout 300 python tools/kbench.py; done
AK_IWARPS=2 timeout 300 python tools/kbench.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log

AK_IMMA=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
grep -E "^E " gpurun_out/pytest_gpu.log | head -5
for im in 0 1; do for iw in 1 2; do echo "imma=$im iw=$iw"; AK_IMMA=$im AK_IWARPS=$iw timeout 300 python tools/kbench.py; done; done
AK_IMMA=1 AK_BATCH3=32 timeout 300 python tools/kbench.py

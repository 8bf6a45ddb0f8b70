timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
grep -E "^E " gpurun_out/pytest_gpu.log | head -3
for s in 1 2; do for b in 16 32; do echo "s=$s b=$b"; AK_SUPERCELL3=$s AK_BATCH3=$b timeout 300 python tools/kbench.py; done; done
echo auto; timeout 300 python tools/kbench.py

timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for b in 16 32; do for s in 2 3; do
  echo "batch=$b"; AK_BATCH3=$b AK_SUPERCELL3=$s timeout 300 python tools/kbench.py
done; done

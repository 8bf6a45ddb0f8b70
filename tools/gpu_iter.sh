timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for iw in 1 2; do for s in 2 3; do
  echo "iwarps=$iw"; AK_IWARPS=$iw AK_SUPERCELL3=$s timeout 300 python tools/kbench.py
done; done
AK_IWARPS=2 timeout 900 python -m pytest tests -m gpu -q -x -k "parity or c4" > gpurun_out/pytest_gpu2.log 2>&1; echo pytest2=$?

set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_kernels.py > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_tile|k_interp3" -s 2 -c 2 -o gpurun_out/prof_r1 python tools/prof_kernels.py > gpurun_out/ncu_full.log 2>&1; echo full=$?
tail -3 gpurun_out/ncu_full.log

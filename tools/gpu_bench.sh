# Round measurement: bench (plain), launch list and full capture of the top kernels (one GPU).
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 1 --quick > gpurun_out/bench_quick.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 300 python tools/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread3|k_interp3" -s 2 -c 2 \
    -o gpurun_out/prof_full python tools/prof_kernels.py > gpurun_out/ncu_full.log 2>&1; echo full=$?

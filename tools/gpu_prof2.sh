timeout 300 python tools/prof_kernels.py > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread3|k_interp3" -s 2 -c 2 -o gpurun_out/prof_r1f python tools/prof_kernels.py > gpurun_out/ncu_full.log 2>&1; echo ncu=$?

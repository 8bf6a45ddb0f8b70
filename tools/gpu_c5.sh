timeout 600 python tools/c5_launches.py > gpurun_out/c5_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_launches.py > gpurun_out/c5_ncu.log 2>&1; echo c5=$?

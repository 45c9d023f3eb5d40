timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/b1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"

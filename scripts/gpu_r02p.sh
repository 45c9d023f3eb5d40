timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02p_c5.json 2> gpurun_out/bench_r02p_c5.err; echo rc=$?
tail -c 3500 gpurun_out/bench_r02p_c5.json; tail -5 gpurun_out/bench_r02p_c5.err
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r02p_c3.json 2> gpurun_out/bench_r02p_c3.err; echo rc=$?
tail -c 1500 gpurun_out/bench_r02p_c3.json; tail -5 gpurun_out/bench_r02p_c3.err

timeout 900 python -m pytest tests -q -m gpu -x -k "nystrom or psd" --durations=5 2>&1 | tail -8
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_r02i_c4.json 2> gpurun_out/bench_r02i_c4.err; echo rc=$?
tail -c 2500 gpurun_out/bench_r02i_c4.json; tail -5 gpurun_out/bench_r02i_c4.err

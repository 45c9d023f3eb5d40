set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "syrk or sketch_space or reduced or c3_full or c2_ or h3" --durations=10 > gpurun_out/pytest_r02c.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_r02c.log
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r02c_c3.json 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench_r02c_c3.json
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r02c_c5.json 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench_r02c_c5.json

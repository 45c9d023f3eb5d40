set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu --durations=25 -rs > gpurun_out/pytest_r02b.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest_r02b.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench rc=$?
tail -3 gpurun_out/bench_r02b.json; tail -20 gpurun_out/bench_r02b.err

timeout 300 python scripts/sketch_probe.py > gpurun_out/sketch_probe.log 2>&1; echo "sketch rc=$?"; tail -9 gpurun_out/sketch_probe.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -15
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c3.log | cut -c1-1200

timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q --timeout 300 -k "jacobi" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_gpu.log | tail -12
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms'])"

timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -25
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench_c3.log

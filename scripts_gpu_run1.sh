set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name(0), torch.cuda.get_device_capability(0))"
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench_c3.log

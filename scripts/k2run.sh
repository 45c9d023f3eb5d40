timeout 300 python scripts/sched_conflicts.py
timeout 300 python scripts/sketch_time.py
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "gather or sketch or srht" 2>&1 | tail -3

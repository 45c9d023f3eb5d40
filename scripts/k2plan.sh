# K2 v2 plan quality (wavefronts per LDS implied by the schedule), K2 time, sketch parity tests
timeout 300 python scripts/sched_conflicts.py
timeout 120 python scripts/sketch_time.py
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "gather or sketch" 2>&1 | tail -3

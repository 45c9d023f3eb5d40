# K2 v3 (paired slices): parity tests, then timing alone at C3 and C5
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "gather or sketch" > $O/k3_tests.log 2>&1; echo tests rc=$?
tail -3 $O/k3_tests.log
timeout 300 python scripts/sketch_time.py 2>&1 | tail -2
timeout 600 python scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -2

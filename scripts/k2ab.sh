# K2: timings at the C5 pass shape and C3, plan quality, the gather tests
O=gpurun_out
{
python scripts/sketch_one.py v2 131072 32768 8000
python scripts/sketch_one.py v2 262144 16384 4000
timeout 300 python scripts/plan_stats.py 32768 8000
timeout 300 python scripts/plan_stats.py 16384 4000
} 2>&1 | tee $O/k2ab.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "gather or sketch or nystrom" 2>&1 | tail -3

O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_reference_api.py -x -q -k "sketch or right or gather or apply" 2>&1 | tail -3
python scripts/right_time.py 2>&1 | tee $O/right_time.txt
python scripts/right_time.py 262144 16384 4000 2>&1 | tee -a $O/right_time.txt

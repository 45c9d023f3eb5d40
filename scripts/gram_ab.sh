O=gpurun_out
for v in old new old new; do cp abtest/libskp_$v.so paper_2605_09755_b200/libskp.so; python scripts/gram_time.py | sed "s/^/$v /"; done 2>&1 | tee $O/gram_ab.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "syrk" 2>&1 | tail -2

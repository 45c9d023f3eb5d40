O=gpurun_out
cp abtest/libskp_old.so paper_2605_09755_b200/libskp.so
python scripts/eig_time.py 520 700 1050 1500 2>&1 | sed 's/^/old /' | tee $O/eig_ab.txt
cp abtest/libskp_new.so paper_2605_09755_b200/libskp.so
python scripts/eig_time.py 520 700 1050 1500 2>&1 | sed 's/^/new /' | tee -a $O/eig_ab.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "eigensolver" 2>&1 | tail -2

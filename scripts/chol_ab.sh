O=gpurun_out
for v in old new old new; do cp abtest/libskp_$v.so paper_2605_09755_b200/libskp.so; python scripts/cholinv_time.py 260 520 1050 | sed "s/^/$v /"; done | tee $O/chol_ab.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "cholinv or cholesky or orth or rank or c2_fp32 or reduced" 2>&1 | tail -2

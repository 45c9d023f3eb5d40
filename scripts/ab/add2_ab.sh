# K2 plan: lanes sorted by their largest per-pass count (T = tree) or by their total (ST, as before)
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "gather or sketch" 2>&1 | tail -2
for rep in 1 2; do for v in T ST; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 600 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1 | sed "s/^/$v alone C5: /"
done; done
for v in T ST; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 300 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 2>&1 | tail -1 | sed "s/^/$v alone C3: /"
  timeout 300 python scripts/ab/run_lib.py $lib scripts/plan_stats.py 32768 8000 2>&1 | tail -4 | sed "s/^/$v plan C5: /"
done

# K2 v3: T = tree (two row buffers), NB3 = three row buffers of 65664 bytes
for v in T NB3; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 300 python scripts/ab/run_lib.py $lib scripts/ab/k2_sum.py 2>&1 | tail -3 | sed "s/^/$v digest: /"
done
for rep in 1 2; do for v in T NB3; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 300 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 2>&1 | tail -1 | sed "s/^/$v alone C3: /"
  timeout 600 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1 | sed "s/^/$v alone C5: /"
done; done

# K2 v3 launched in row chunks of R row steps per CTA (a kernel boundary re-aligns the CTAs of a row group): T = one launch per pass
O=gpurun_out
for v in T CH128 CH512 CH2048; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 300 python scripts/ab/run_lib.py $lib scripts/ab/k2_sum.py 2>&1 | tail -1 | sed "s/^/$v digest: /"
  timeout 300 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 2>&1 | tail -1 | sed "s/^/$v alone C3: /"
  timeout 600 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1 | sed "s/^/$v alone C5: /"
done

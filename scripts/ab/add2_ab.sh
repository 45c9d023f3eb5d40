for rep in 1 2; do for v in CH384 CH768 CH1024; do
  lib=scripts/ab/libskp_$v.so
  timeout 600 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1 | sed "s/^/$v alone C5: /"
done; done

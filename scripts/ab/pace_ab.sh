# K2 row pacing A/B: P = paced (the tree's libskp.so), B = unpaced variant (scripts/ab/libskp_B.so)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "gather or sketch" 2>&1 | tail -2
for v in P B; do
  lib=paper_2605_09755_b200/libskp.so; [ $v = B ] && lib=scripts/ab/libskp_B.so
  timeout 300 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 2>&1 | tail -1 | sed "s/^/$v alone C3: /"
  timeout 600 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1 | sed "s/^/$v alone C5: /"
done
for v in P B; do
  lib=paper_2605_09755_b200/libskp.so; [ $v = B ] && lib=scripts/ab/libskp_B.so
  timeout 600 python scripts/ab/run_lib.py $lib bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu > $O/pace_c3_$v.json 2>/dev/null
  timeout 900 python scripts/ab/run_lib.py $lib bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/pace_c5_$v.json 2>/dev/null
  for c in c3 c5; do python -c "
import json; d=json.loads(open('$O/pace_${c}_$v.json').read().strip().splitlines()[-1])
print('$v $c', d['value'], d['phases_ms']['apply_right'], {k: round(v['ms_per_launch'],2) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])"; done
done
for v in P B; do
  lib=paper_2605_09755_b200/libskp.so; [ $v = B ] && lib=scripts/ab/libskp_B.so
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pair -s 4 -c 2 --csv --log-file $O/pace_ncu_$v.csv python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 > /dev/null 2>&1
  grep -E "dram__bytes|duration|hit_rate" $O/pace_ncu_$v.csv | awk -F'","' '{print "'$v' ncu C5:", $(NF-3), $(NF-2), $(NF-1), $NF}'
done

# K2 row chain: alone timings at C3 and C5 shapes, DRAM bytes of the tree's variant
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "gather or sketch" 2>&1 | tail -2
for v in T B W2 W8 W4L2; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 300 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 2>&1 | tail -1 | sed "s/^/$v alone C3: /"
  timeout 600 python scripts/ab/run_lib.py $lib scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1 | sed "s/^/$v alone C5: /"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pair -s 4 -c 2 --csv --log-file $O/chain_ncu_T.csv python scripts/sketch_time.py 1048576 32768 8000 > /dev/null 2>&1
grep -E "dram__bytes|duration|hit_rate" $O/chain_ncu_T.csv | awk -F'","' '{print "T ncu C5:", $(NF-3), $(NF-2), $(NF-1), $NF}'

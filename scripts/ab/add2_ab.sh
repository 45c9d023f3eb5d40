# K2: T = tree, H = HEAD: C4 (K2 v2, fp64 accumulation, several column passes) and C5 in the step
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "gather or sketch" 2>&1 | tail -2
for v in T H; do
  lib=scripts/ab/libskp_$v.so; [ $v = T ] && lib=paper_2605_09755_b200/libskp.so
  timeout 600 python scripts/ab/run_lib.py $lib bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/pf_c4_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/pf_c4_$v.json').read().strip().splitlines()[-1])
print('$v c4', d['value'], d.get('phases_ms'), d['roofline'].get('ms_per_launch'))"
  timeout 900 python scripts/ab/run_lib.py $lib bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/pf_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/pf_c5_$v.json').read().strip().splitlines()[-1])
print('$v c5', d['value'], d['phases_ms']['apply_right'], {k: round(v['ms_per_launch'],2) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done

# A: pair + hint, B: pair no hint, C: old + hint, D: old no hint
O=gpurun_out
for v in A B C D; do
  timeout 300 python scripts/ab/run_lib.py scripts/ab/libskp_$v.so scripts/sketch_time.py 2>&1 | tail -1 | sed "s/^/$v alone: /"
  timeout 600 python scripts/ab/run_lib.py scripts/ab/libskp_$v.so bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu > $O/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/ab_$v.json').read().strip().splitlines()[-1])
print('$v C3', d['value'], d['phases_ms']['apply_right'], {k: round(v['ms_per_launch'],2) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
for v in A C D; do
  timeout 900 python scripts/ab/run_lib.py scripts/ab/libskp_$v.so bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ab5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/ab5_$v.json').read().strip().splitlines()[-1])
print('$v C5', d['value'], d['phases_ms']['apply_right'], {k: round(v['ms_per_launch'],2) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done

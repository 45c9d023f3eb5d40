# K2 A/B at full C5 (bench's live kernel timing), old vs new libskp, alternating
O=gpurun_out
: > $O/k2_ab_full.txt
for v in old new old new; do
  cp abtest/libskp_$v.so paper_2605_09755_b200/libskp.so
  timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/k2ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/k2ab_$v.json').read().strip().splitlines()[-1])
print('$v', 'step', d['value'], 'sketch', d['kernels']['sketch']['ms_per_launch'], 'apply_right', d['phases_ms']['apply_right'], d['clocks']['sm_mhz'])" >> $O/k2_ab_full.txt
done
cat $O/k2_ab_full.txt

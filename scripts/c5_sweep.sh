# BASELINE configs[4]: the l x q sweep of C5 on one B200 (device-timed rSVD per step)
O=gpurun_out
: > $O/c5_sweep.txt
for l in 4000 8000 16000; do for q in 1 2 4; do
  timeout 900 python bench.py --l $l --q $q --steps 2 --warmup 1 --no-cpu --no-e2e > $O/sweep_${l}_${q}.json 2> $O/sweep_${l}_${q}.err
  python -c "
import json; d=json.loads(open('$O/sweep_${l}_${q}.json').read().strip().splitlines()[-1])
print('l=$l q=$q', d['value'], 'ms', d['phases_ms'], d['power_path'][:40], 'rel_err %.5f' % d['rel_err'], d['clocks']['sm_mhz'])" >> $O/c5_sweep.txt 2>&1
done; done
cat $O/c5_sweep.txt

O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_api.py -x -q 2>&1 | tail -2
: > $O/c5_sweep2.txt
for lq in "4000 1" "8000 2"; do set -- $lq; l=$1; q=$2
  timeout 900 python bench.py --l $l --q $q --steps 2 --warmup 1 --no-cpu --no-e2e > $O/sweep_${l}_${q}.json 2> $O/sweep_${l}_${q}.err
  python -c "
import json; d=json.loads(open('$O/sweep_${l}_${q}.json').read().strip().splitlines()[-1])
print('l=$l q=$q', d['value'], 'ms', d['phases_ms'], d['power_path'][:40], 'rel_err %.5f' % d['rel_err'], d['clocks']['sm_mhz'])" >> $O/c5_sweep2.txt 2>&1
done
cat $O/c5_sweep2.txt
timeout 900 python scripts/randsvd_probe.py C5 > $O/probe_c5.txt 2>&1; tail -25 $O/probe_c5.txt

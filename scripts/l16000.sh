# C5 at l = 16000 on one B200: the blocked range finder (A~ does not fit beside A)
O=gpurun_out
timeout 1500 python bench.py --l 16000 --steps 2 --warmup 1 --no-cpu > $O/bench_c5_l16000.json 2> $O/bench_c5_l16000.err; echo rc=$?
tail -3 $O/bench_c5_l16000.err
python -c "import json; d=json.loads(open('$O/bench_c5_l16000.json').read().strip().splitlines()[-1]); print(d['value'], d['phases_ms'], d.get('power_path'), (d.get('e2e') or {}).get('value'), d['clocks'], d['rel_err'])"

O=gpurun_out
timeout 2000 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench_c5_k6.json 2> $O/bench_c5_k6.err; echo c5 rc=$?
python -c "import json; d=json.loads(open('$O/bench_c5_k6.json').read().strip().splitlines()[-1]); print(d['value'], d.get('phases_ms'), (d.get('e2e') or {}).get('value'), d['clocks'])"
timeout 900 python scripts/randsvd_probe.py C5 2>&1 | grep -E "eig_desc|gram64|chol|^\{"

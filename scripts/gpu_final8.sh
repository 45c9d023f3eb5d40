# round-end evidence (r02zg): smoke, GPU tests, C5/C3 bench lines
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -q -m gpu --durations=5 > $O/pytest_final.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_final.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_final_c5.json 2> $O/bench_final_c5.err; echo c5 rc=$?
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 > $O/bench_final_c3.json 2> $O/bench_final_c3.err; echo c3 rc=$?
for c in c5 c3; do python -c "import json; d=json.loads(open('$O/bench_final_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d.get('phases_ms'), (d.get('e2e') or {}).get('value'), d['clocks'], d['gpu_launches'])"; done

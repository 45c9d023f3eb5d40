# round-end evidence: GPU tests, the C5 / C3 / C4 bench lines, launch lists
O=gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_final.log 2>&1; echo pytest rc=$?
tail -4 $O/pytest_final.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_final_c5.json 2> $O/bench_final_c5.err; echo c5 rc=$?
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 > $O/bench_final_c3.json 2> $O/bench_final_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 > $O/bench_final_c4.json 2> $O/bench_final_c4.err; echo c4 rc=$?
for c in c5 c3 c4; do python -c "import json; d=json.loads(open('$O/bench_final_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d.get('phases_ms'), (d.get('e2e') or {}).get('value'), d['clocks'])"; done

# re-entry check (r02za): smoke, GPU tests, C5 bench line
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -q -m gpu -x --durations=5 > $O/r02za_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/r02za_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/r02za_bench_c5.json 2> $O/r02za_bench_c5.err; echo c5 rc=$?
python -c "import json; d=json.loads(open('$O/r02za_bench_c5.json').read().strip().splitlines()[-1]); print(d['value'], d.get('phases_ms'), (d.get('e2e') or {}).get('value'), d['clocks'])"

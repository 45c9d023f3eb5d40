# round-end evidence (r02zf): smoke, GPU tests, C5/C3/C4 bench lines, C5 launch list
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_final.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_final.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_final_c5.json 2> $O/bench_final_c5.err; echo c5 rc=$?
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 > $O/bench_final_c3.json 2> $O/bench_final_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 > $O/bench_final_c4.json 2> $O/bench_final_c4.err; echo c4 rc=$?
for c in c5 c3 c4; do python -c "import json; d=json.loads(open('$O/bench_final_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d.get('phases_ms'), (d.get('e2e') or {}).get('value'), d['clocks'])"; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:skp:: -c 400 --csv --log-file $O/r02zf_c5_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo ncu rc=$?
python scripts/summarize_ncu.py launches $O/r02zf_c5_launches.csv $O/r02zf_launches_c5.txt; head -12 $O/r02zf_launches_c5.txt

# round-end evidence (r02x): GPU tests, C5/C3/C4 bench lines, reference arm (C3), 2 gloo ranks
# on one GPU through bench.py, C5 launch list
O=gpurun_out
timeout 2000 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_final.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_final.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_final_c5.json 2> $O/bench_final_c5.err; echo c5 rc=$?
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 > $O/bench_final_c3.json 2> $O/bench_final_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 > $O/bench_final_c4.json 2> $O/bench_final_c4.err; echo c4 rc=$?
for c in c5 c3 c4; do python -c "import json; d=json.loads(open('$O/bench_final_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d.get('phases_ms'), (d.get('e2e') or {}).get('value'), d['clocks'])"; done
timeout 900 python bench.py --impl reference --config C3 --steps 1 --warmup 0 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err; echo ref rc=$?; tail -c 600 $O/bench_ref_c3.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C3 --dist-backend gloo --steps 2 --warmup 1 --no-cpu > $O/bench_2rank_c3.json 2> $O/bench_2rank_c3.err; echo 2rank rc=$?; tail -c 400 $O/bench_2rank_c3.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/r02x_c5_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo ncu rc=$?
python scripts/summarize_ncu.py launches $O/r02x_c5_launches.csv $O/r02x_launches_c5_1step.txt; head -25 $O/r02x_launches_c5_1step.txt

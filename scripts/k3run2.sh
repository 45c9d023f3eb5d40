# hinted mbarrier waits + K2 v3: kernel tests, K2 alone at C3/C5, C5 and C3 bench lines
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > $O/k3b_tests.log 2>&1; echo tests rc=$?
tail -2 $O/k3b_tests.log
timeout 300 python scripts/sketch_time.py 2>&1 | tail -1
timeout 600 python scripts/sketch_time.py 1048576 32768 8000 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/k3b_bench_c5.json 2> $O/k3b_bench_c5.err; echo c5 rc=$?
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu > $O/k3b_bench_c3.json 2> $O/k3b_bench_c3.err; echo c3 rc=$?
for c in c5 c3; do python -c "
import json; d=json.loads(open('$O/k3b_bench_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d.get('phases_ms'), d['clocks']['sm_mhz'])
print({k: round(v['ms_per_launch'],2) for k, v in d['kernels'].items()})"; done

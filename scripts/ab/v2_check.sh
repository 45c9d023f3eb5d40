# K2 v2 (atom.inc): kernel tests, Nystrom tests, C4 bench
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/v2_c4.json 2>/dev/null
python -c "
import json; d=json.loads(open('$O/v2_c4.json').read().strip().splitlines()[-1])
print('c4', d['value'], d['roofline'].get('ms_per_launch'))"

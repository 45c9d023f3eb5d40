#!/bin/bash
# Round evidence on one B200 (run under gpurun):  bash scripts/profile_round.sh TAG
#   1. GPU tests, 2. the bench line, 3. the launch list of the same bench
#   command (metrics-only ncu pass), 4. ncu --set full of the two hot kernels
#   (each command first ran clean without ncu).
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"
tail -3 $O/${TAG}_pytest.log
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench rc=$?"
cat $O/${TAG}_bench.json
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_bench_short.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > $O/${TAG}_ncu_launch.log 2>&1
echo "launch-list rc=$?"
python scripts/gemm_one.py nn h3 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:gemm_h3_kernel -s 2 -c 1 \
    -o $O/${TAG}_gemm_h3_nn -f python scripts/gemm_one.py nn h3 > $O/${TAG}_ncu_gemm.log 2>&1
echo "ncu gemm rc=$?"
python scripts/gemm_one.py qta h3s > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:gemm_h3s_kernel -s 1 -c 1 \
    -o $O/${TAG}_gemm_h3s_qta -f python scripts/gemm_one.py qta h3s > $O/${TAG}_ncu_h3s.log 2>&1
echo "ncu h3s rc=$?"
python scripts/sketch_one.py v2 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:sketch_gather_kernel -s 1 -c 1 \
    -o $O/${TAG}_sketch_gather -f python scripts/sketch_one.py v2 > $O/${TAG}_ncu_sketch.log 2>&1
echo "ncu sketch rc=$?"

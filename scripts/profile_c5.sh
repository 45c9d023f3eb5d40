#!/bin/bash
# C5 evidence on one B200 (run under gpurun):  bash scripts/profile_c5.sh TAG
#   1. launch list of one bench step (metrics-only ncu pass; the command first ran clean)
#   2. ncu --set full of the power GEMM (K4h), randsvd's A^T Q (K4s) and the sketch (K2)
#      at C5 shapes (scripts/gemm_one.py / sketch_one.py ran clean first)
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > $O/${TAG}_c5_short.json 2>&1 || { tail $O/${TAG}_c5_short.json; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_c5_launches.csv python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu \
    > $O/${TAG}_c5_ncu_launch.log 2>&1
echo "launch-list rc=$?"
for spec in "nn h3 gemm_h3_kernel 2" "qta h3s gemm_h3s_kernel 1"; do
  set -- $spec
  python scripts/gemm_one.py $1 $2 3 C5 > /dev/null && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
      -o $O/${TAG}_c5_$2_$1 -f python scripts/gemm_one.py $1 $2 3 C5 > $O/${TAG}_c5_ncu_$2_$1.log 2>&1
  echo "ncu $2 $1 rc=$?"
done
python scripts/sketch_one.py v2 1048576 32768 8000 > /dev/null && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sketch_gather_kernel -s 1 -c 1 \
    -o $O/${TAG}_c5_sketch_gather -f python scripts/sketch_one.py v2 1048576 32768 8000 > $O/${TAG}_c5_ncu_sketch.log 2>&1
echo "ncu sketch rc=$?"

O=gpurun_out
for spec in "qta h3s gemm_h3s_kernel C5" "syrk h3 gemm_h3_kernel C5" "nn h3 gemm_h3_kernel C5" "qta h3s gemm_h3s_kernel C3" "syrk h3 gemm_h3_kernel C3" "nn h3 gemm_h3_kernel C3"; do
  set -- $spec
  python scripts/gemm_one.py $1 $2 1 $4 > /dev/null || continue
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $O/r02v_$4_$1 -f python scripts/gemm_one.py $1 $2 1 $4 > $O/r02v_ncu_$4_$1.log 2>&1
  echo "$4 $1 rc=$?"
done

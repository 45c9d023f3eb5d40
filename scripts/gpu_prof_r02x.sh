# ncu --set full of randsvd's B^T = A^T Q (K4s, 8 split warps) at C5 and C3
O=gpurun_out
for spec in "qta h3s gemm_h3s_kernel C5" "qta h3s gemm_h3s_kernel C3"; do
  set -- $spec
  python scripts/gemm_one.py $1 $2 1 $4 > /dev/null || continue
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $O/r02x_$4_$1 -f python scripts/gemm_one.py $1 $2 1 $4 > $O/r02x_ncu_$4_$1.log 2>&1
  echo "$4 $1 rc=$?"
  python scripts/summarize_ncu.py full $O/r02x_$4_$1.ncu-rep $O/r02x_$4_$1_full.txt
done

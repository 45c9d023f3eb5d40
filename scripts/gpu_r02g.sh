O=gpurun_out
python scripts/gemm_one.py syrk h3 3 C5
python scripts/gemm_one.py qta h3s 3 C5
python scripts/gemm_one.py syrk h3 3 C3
python scripts/gemm_one.py qta h3s 3 C3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_h3_kernel -s 1 -c 1 -o $O/r02g_c5_syrk -f python scripts/gemm_one.py syrk h3 1 C5 > $O/r02g_ncu_syrk.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_h3s_kernel -s 1 -c 1 -o $O/r02g_c5_h3s_qta -f python scripts/gemm_one.py qta h3s 1 C5 > $O/r02g_ncu_qta.log 2>&1; echo rc=$?

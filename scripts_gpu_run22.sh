python scripts/gemm_one.py nn > gpurun_out/g1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/gemm_nn2 python scripts/gemm_one.py nn > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?"

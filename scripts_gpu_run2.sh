timeout 240 python scripts/gemm_probe.py > gpurun_out/gemm_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/gemm_probe.log | tail -45

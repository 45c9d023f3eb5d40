timeout 300 python scripts/sketch_probe.py > gpurun_out/sketch_probe.log 2>&1; echo "sketch rc=$?"; cat gpurun_out/sketch_probe.log | tail -12
SKP_SKETCH_SLAB=1 timeout 300 python scripts/sketch_probe.py 2>&1 | tail -3

python scripts/sketch_one.py > gpurun_out/s1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_rows -s 1 -c 1 -o gpurun_out/sketch_rows2 python scripts/sketch_one.py > gpurun_out/ncu_sketch.log 2>&1; echo "ncu rc=$?"

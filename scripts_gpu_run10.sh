python scripts/sketch_one.py > gpurun_out/s1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_rows -s 1 -c 1 -o gpurun_out/sketch_rows python scripts/sketch_one.py > gpurun_out/ncu_sketch.log 2>&1; echo "ncu rc=$?"
python scripts/sketch_one.py > gpurun_out/s1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sketch.csv python scripts/sketch_one.py > /dev/null 2>&1; echo "ncu2 rc=$?"

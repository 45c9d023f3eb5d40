O=gpurun_out
python scripts/sketch_one.py v2 1048576 32768 8000 > /dev/null && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_gather_kernel -s 2 -c 1 -o $O/r02k_c5_sketch_gather -f python scripts/sketch_one.py v2 1048576 32768 8000 > $O/r02k_ncu_c5.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_gather_kernel -s 2 -c 1 -o $O/r02k_c3_sketch_gather -f python scripts/sketch_one.py v2 262144 16384 4000 > $O/r02k_ncu_c3.log 2>&1; echo rc=$?

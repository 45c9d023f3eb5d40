O=gpurun_out
python scripts/sketch_one.py v2 131072 32768 8000 | tee $O/k2prev.txt
python scripts/sketch_one.py v2 262144 16384 4000 | tee -a $O/k2prev.txt
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sketch_gather_kernel -s 2 -c 2 --csv python scripts/sketch_one.py v2 131072 32768 8000 2>&1 | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print $1, $(NF-2), $NF}' | tee -a $O/k2prev.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "gather or sketch or nystrom or right" 2>&1 | tail -2

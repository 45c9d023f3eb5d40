O=gpurun_out
python scripts/sketch_one.py v2 131072 32768 8000 > $O/k2_c5like.txt 2>&1
cat $O/k2_c5like.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sketch_gather_kernel -s 2 -c 1 -o $O/k2_c5like -f python scripts/sketch_one.py v2 131072 32768 8000 > $O/k2_ncu.log 2>&1
tail -3 $O/k2_ncu.log

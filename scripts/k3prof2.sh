# K2 v3 (packed adds) ncu captures: C3 (one launch) and C5 (one pass)
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair -s 2 -c 1 -o $O/r02zd_c3_pair python scripts/sketch_time.py > $O/k3_ncu_c3.log 2>&1; echo ncu3 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair -s 4 -c 2 -o $O/r02zd_c5_pair python scripts/sketch_time.py 1048576 32768 8000 > $O/k3_ncu_c5.log 2>&1; echo ncu5 rc=$?

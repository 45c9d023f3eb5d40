python scripts/one_step.py C5 > gpurun_out/r02e_c5_step.txt 2>&1 || exit 1
cat gpurun_out/r02e_c5_step.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_c5_launches.csv python scripts/one_step.py C5 > gpurun_out/r02e_c5_ncu.log 2>&1
echo ncu rc=$?
python scripts/one_step.py C3 > gpurun_out/r02e_c3_step.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_c3_launches.csv python scripts/one_step.py C3 > gpurun_out/r02e_c3_ncu.log 2>&1
echo ncu rc=$?

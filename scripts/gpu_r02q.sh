timeout 900 python -m pytest tests -q -m gpu -x -k "syrk or h3s or h3 or c2_bench or sketch_space" 2>&1 | tail -3
python scripts/gemm_one.py syrk h3 3 C5
python scripts/gemm_one.py qta h3s 3 C5
python scripts/gemm_one.py syrk h3 3 C3
python scripts/gemm_one.py qta h3s 3 C3
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_h3 -c 2 python scripts/gemm_one.py qta h3s 1 C5 2>&1 | grep -E "dram__|duration|per_second" 
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_h3 -c 2 python scripts/gemm_one.py syrk h3 1 C5 2>&1 | grep -E "dram__|duration|per_second"

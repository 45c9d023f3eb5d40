python scripts/plan_stats.py 16384 4000 | tail -1
python scripts/plan_stats.py 32768 8000 | tail -1
python scripts/sketch_one.py v2 262144 16384 4000
python scripts/sketch_one.py v2 1048576 32768 8000
python scripts/sketch_one.py v2 65536 65536 4096
timeout 600 python -m pytest tests -q -m gpu -x -k "gather or sketch" 2>&1 | tail -2

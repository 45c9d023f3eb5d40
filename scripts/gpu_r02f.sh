timeout 600 python -m pytest tests -q -m gpu -x -k "syrk or sketch_space or h3" 2>&1 | tail -4
python scripts/one_step.py C5 2>&1 | tail -2
python scripts/one_step.py C3 2>&1 | tail -2

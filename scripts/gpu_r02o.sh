timeout 900 python -m pytest tests -q -m gpu -x -k "syrk or emit or h3 or c2_ or reduced or sketch_space or planes or rank_kept" 2>&1 | tail -4
python scripts/one_step.py C5 2>&1 | tail -1
python scripts/one_step.py C3 2>&1 | tail -1

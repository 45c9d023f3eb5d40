timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_r02h.log 2>&1; echo pytest rc=$?
tail -22 gpurun_out/pytest_r02h.log
bash scripts/sanitize.sh

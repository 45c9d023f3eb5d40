set -x
free -g; nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_r02a.log 2>&1; echo rc=$?
tail -30 gpurun_out/pytest_r02a.log

timeout 600 python bench.py --config C2 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/c2_1.log 2>&1; echo "1rank rc=$?"
tail -1 gpurun_out/c2_1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['rel_err'], d['sigma_1'], d['n_gpus'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config C2 --steps 2 --warmup 1 --no-cpu --dist-backend gloo > gpurun_out/c2_2.log 2>&1; echo "2rank rc=$?"
grep metric gpurun_out/c2_2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['rel_err'], d['sigma_1'], d['n_gpus'], d['e2e'])"
tail -3 gpurun_out/c2_2.log

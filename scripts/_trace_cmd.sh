cd $GRAFT_REPO_ROOT
SS_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 --layers 2 > gpurun_out/tp2.log 2>&1; echo rc=$?
grep -E "Error|error" gpurun_out/tp2.log | head -5; grep '^{' gpurun_out/tp2.log | cut -c1-700
SS_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 3 --warmup 3 --e2e-steps 2 --layers 2 > gpurun_out/tp4.log 2>&1; echo rc=$?
grep -E "Error|error" gpurun_out/tp4.log | head -5; grep '^{' gpurun_out/tp4.log | cut -c1-300

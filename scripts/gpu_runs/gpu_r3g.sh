cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/r3g_mgpu.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r3g_mgpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus $NG --steps 100 --warmup 5 > gpurun_out/r3g_bench_n$NG.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus $NG --workload c3 --steps 100 --warmup 5 --no-e2e > gpurun_out/r3g_c3_n$NG.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/r2j_mgpu_$NG.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r2j_mgpu_$NG.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $NG --steps 100 --warmup 5 > gpurun_out/r2j_bench_n$NG.log 2>&1
echo "bench exit $?" >> gpurun_out/r2j_bench_n$NG.log
TMD_TRACE_REBUILD=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus $NG --steps 60 --warmup 5 --no-e2e > gpurun_out/r2j_bench_trace_n$NG.log 2>&1

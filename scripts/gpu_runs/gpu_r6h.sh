cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/r6h_mgpu_$NG.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r6h_mgpu_$NG.log
timeout 900 python bench.py --gpus $NG --steps 100 --warmup 5 > gpurun_out/r6h_bench_n$NG.log 2>&1; echo "rc $?" >> gpurun_out/r6h_bench_n$NG.log

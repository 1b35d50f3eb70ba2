cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/r2r_mgpu_$NG.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r2r_mgpu_$NG.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "torchrun or two_ranks" > gpurun_out/r2r_pytest_multi.log 2>&1
for n in 2 $NG; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 100 --warmup 5 > gpurun_out/r2r_bench_n$n.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2r_bench20_n$n.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --workload c3 --steps 100 --warmup 5 --no-e2e > gpurun_out/r2r_bench_c3_n$n.log 2>&1
done
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2r_bench_c3_n1.log 2>&1

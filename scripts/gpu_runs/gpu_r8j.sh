cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r8j_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r8j_pytest_gpu.log
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r8j_bench_weak_n1.log 2>&1
for n in 4 8; do
  if [ "$NG" -ge $n ]; then
    timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $n scripts/mgpu_check.py > gpurun_out/mgpu_$n.log 2>&1
    echo "mgpu exit $?" >> gpurun_out/mgpu_$n.log
  fi
done
for n in 2 4 8; do
  if [ "$NG" -ge $n ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 100 --warmup 5 > gpurun_out/bench_weak_n$n.log 2>&1
    echo "bench exit $?" >> gpurun_out/bench_weak_n$n.log
  fi
done
echo done

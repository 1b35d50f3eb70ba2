cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r8n_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r8n_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/r8n_pytest_gpu.log
for n in 2 4; do
  if [ "$NG" -ge $n ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n scripts/mgpu_check.py > gpurun_out/r8n_mgpu_$n.log 2>&1
    echo "mgpu $n rc $?"
  fi
done
timeout 900 python bench.py > gpurun_out/r8n_bench_n1.log 2>&1; echo "bench 1 rc $?"
for n in 2 4; do
  if [ "$NG" -ge $n ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n > gpurun_out/r8n_bench_n$n.log 2>&1
    echo "bench $n rc $?"
  fi
done
timeout 900 python bench.py --impl reference > gpurun_out/r8n_bench_ref.log 2>&1; echo "ref rc $?"
for n in 1 2 4; do
  if [ "$NG" -ge $n ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n --workload c3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/r8n_c3_n$n.log 2>&1
    echo "c3 $n rc $?"
  fi
done

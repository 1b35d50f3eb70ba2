cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/bench_c5_1.log 2>&1
echo "c5 rc $?"
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --workload c5 --no-e2e > gpurun_out/bench_c5_2.log 2>&1
echo "c5 2 rc $?"

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke rc $?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
timeout 600 torchrun --standalone --nproc-per-node 4 scripts/mgpu_check.py > gpurun_out/mgpu4.log 2>&1
echo "mgpu4 rc $?"
timeout 600 torchrun --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/mgpu2.log 2>&1
echo "mgpu2 rc $?"
timeout 300 python bench.py > gpurun_out/bench1.log 2>&1
echo "bench1 rc $?"
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/bench2.log 2>&1
echo "bench2 rc $?"
timeout 300 torchrun --standalone --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/bench4.log 2>&1
echo "bench4 rc $?"
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref1.log 2>&1
echo "ref1 rc $?"
for n in 1 2 4; do
timeout 300 torchrun --standalone --nproc-per-node $n bench.py --gpus $n --workload c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_$n.log 2>&1
echo "c3 $n rc $?"
done

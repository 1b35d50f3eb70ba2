cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 torchrun --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/mgpu2.log 2>&1
echo "mgpu2 rc $?"
timeout 600 torchrun --standalone --nproc-per-node 4 scripts/mgpu_check.py > gpurun_out/mgpu4.log 2>&1
echo "mgpu4 rc $?"
for i in 1 2; do
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-e2e > gpurun_out/bench2_$i.log 2>&1
timeout 300 torchrun --standalone --nproc-per-node 4 bench.py --gpus 4 --no-e2e > gpurun_out/bench4_$i.log 2>&1
done

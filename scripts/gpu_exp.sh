cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
timeout 300 torchrun --standalone --nproc-per-node 4 bench.py --gpus 4 --no-e2e > gpurun_out/bench4_$i.log 2>&1
echo "bench4 rc $?"
done

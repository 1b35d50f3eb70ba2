cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --steps 100 --warmup 5 --no-e2e > gpurun_out/bench2c_$i.log 2>&1
done

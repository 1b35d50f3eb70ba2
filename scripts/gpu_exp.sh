cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1_$i.log 2>&1
done
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/bench2.log 2>&1

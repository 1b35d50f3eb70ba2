cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6 7 8; do
TMD_TRACE_REBUILD=3 timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-e2e > gpurun_out/bench2_$i.log 2>&1
mkdir -p gpurun_out/tr$i; mv gpurun_out/rebuild_trace_rank*.json gpurun_out/tr$i/ 2>/dev/null
echo "bench2 rc $?"
done

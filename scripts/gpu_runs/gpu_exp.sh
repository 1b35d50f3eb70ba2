# Ad-hoc experiment runner for gpurun (edit freely):
#   /usr/local/graft/bin/gpurun --gpus 4 --timeout 1500 -- 'bash scripts/gpu_exp.sh'
# Example: repeated multi-GPU bench runs, epoch times per run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-e2e > gpurun_out/bench2_$i.log 2>&1
timeout 300 torchrun --standalone --nproc-per-node 4 bench.py --gpus 4 --no-e2e > gpurun_out/bench4_$i.log 2>&1
done

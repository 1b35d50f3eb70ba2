cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "0 4" "1 4" "1 2" "1 6" "1 0"; do set -- $cfg
TMD_OVERLAP=$1 TMD_RANGE_BLOCKS_PER_SM=$2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2966$2 bench.py --gpus 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3s_n2_ov$1_b$2.log 2>&1
done

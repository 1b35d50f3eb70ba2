cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/diag_mgpu.py 80 > gpurun_out/diag_1.log 2>&1
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/diag_mgpu.py 80 > gpurun_out/diag_2.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/profile_rebuild_mgpu.py 80 > gpurun_out/r3i_rebuild_p2.log 2>&1

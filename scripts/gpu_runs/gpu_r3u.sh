cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 4 scripts/profile_rebuild_mgpu.py 32 > gpurun_out/r3u_rebuild_p4_c32.log 2>&1

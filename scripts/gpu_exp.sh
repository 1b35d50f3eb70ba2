cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 torchrun --standalone --nproc-per-node 2 scripts/host_epoch.py 80 > gpurun_out/host_epoch2.log 2>&1
echo "rc $?"

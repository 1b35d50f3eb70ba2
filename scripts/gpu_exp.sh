cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/profile_epoch.py --cells 80 > gpurun_out/epoch_weak.log 2>&1
timeout 600 python scripts/profile_epoch.py --cells 32 > gpurun_out/epoch_c2.log 2>&1
echo done

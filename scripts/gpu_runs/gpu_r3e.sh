cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/profile_window.py c5 > gpurun_out/r3e_win_c5.log 2>&1
TMD_EPOCH_SYNC=1 timeout 300 python scripts/profile_window.py c5 > gpurun_out/r3e_win_c5sync.log 2>&1

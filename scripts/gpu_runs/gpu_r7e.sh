cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/profile_window.py c5 > gpurun_out/r7e_win_c5.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/diag_steps.py 80 45 > gpurun_out/diag_steps.log 2>&1
echo done

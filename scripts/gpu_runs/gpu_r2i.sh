cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/experiments/exp_smem2.py 80 70 > gpurun_out/r2i_exp_smem2.log 2>&1

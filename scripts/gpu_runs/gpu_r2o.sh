cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/r2o_ab python scripts/experiments/exp_ab.py > gpurun_out/r2o_ab.log 2>&1

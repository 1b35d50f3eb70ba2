cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/r6f_relaunch.log 2>&1; echo "rc $?" >> gpurun_out/r6f_relaunch.log

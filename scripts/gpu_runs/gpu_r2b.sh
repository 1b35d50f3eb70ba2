cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/experiments/exp_step3.py 80 70 > gpurun_out/r2b_exp_step3.log 2>&1
timeout 900 python -m pytest tests/test_loopback_gpu.py -x -q > gpurun_out/r2b_loopback.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_loopback.log

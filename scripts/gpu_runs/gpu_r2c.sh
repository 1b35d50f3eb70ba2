cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/experiments/exp_step4.py 80 70 > gpurun_out/r2c_exp_step4.log 2>&1
timeout 900 python -m pytest tests/test_loopback_gpu.py -x -q > gpurun_out/r2c_loopback.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_loopback.log

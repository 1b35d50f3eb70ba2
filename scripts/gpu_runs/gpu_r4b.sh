cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_loopback_gpu.py -x -q > gpurun_out/r4b_loop_g1_$i.log 2>&1; tail -1 gpurun_out/r4b_loop_g1_$i.log
TMD_MAIL_GATHER=0 timeout 900 python -m pytest tests/test_loopback_gpu.py -x -q > gpurun_out/r4b_loop_g0_$i.log 2>&1; tail -1 gpurun_out/r4b_loop_g0_$i.log
done

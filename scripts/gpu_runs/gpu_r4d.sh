cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python scripts/stress_allgather.py 8 1000 > gpurun_out/r4d_stress.log 2>&1
timeout 300 python scripts/stress_allgather.py 8 1000 >> gpurun_out/r4d_stress.log 2>&1
for i in 1 2 3 4; do
timeout 900 python -m pytest tests/test_loopback_gpu.py -q > gpurun_out/r4d_loop_$i.log 2>&1; tail -1 gpurun_out/r4d_loop_$i.log
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r4d_pytest.log 2>&1; tail -1 gpurun_out/r4d_pytest.log

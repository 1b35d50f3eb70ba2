cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/stress_allgather.py 8 500 > gpurun_out/r4c_stress.log 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python scripts/stress_allgather.py 8 500 >> gpurun_out/r4c_stress.log 2>&1

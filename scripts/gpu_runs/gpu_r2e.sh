cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r2e_fp64_peak.json 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_smem scripts/experiments/exp_smem.cu && /tmp/exp_smem > gpurun_out/r2e_exp_smem.log 2>&1
timeout 600 python -m pytest tests/test_loopback_gpu.py -x -q -k capacity > gpurun_out/r2e_cap.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/debug_build.py > gpurun_out/dbg.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "split or golden_cells or step_kernel" > gpurun_out/dbg_pytest.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "odd_boxes" > gpurun_out/r6j_pytest.log 2>&1; tail -3 gpurun_out/r6j_pytest.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r5e_pytest.log 2>&1; tail -1 gpurun_out/r5e_pytest.log

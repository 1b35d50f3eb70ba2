cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/profile_rebuild.py 40 sd > gpurun_out/r2v_rebuild_c5.log 2>&1
timeout 300 python scripts/profile_rebuild.py 80 > gpurun_out/r2v_rebuild_lj80.log 2>&1
timeout 300 python scripts/profile_epoch_host.py > gpurun_out/r2v_epoch_host.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2v_pytest.log 2>&1

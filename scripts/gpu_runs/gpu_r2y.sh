cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_pytest.log 2>&1
timeout 300 python scripts/profile_rebuild.py 80 > gpurun_out/r2y_rebuild_lj80.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r2y_bench.log 2>&1

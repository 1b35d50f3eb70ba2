cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2z_pytest.log 2>&1
for v in 0 1; do TMD_BUILD_VARIANT=$v timeout 300 python scripts/profile_rebuild.py 80 > gpurun_out/r2z_rebuild_lj80_v$v.log 2>&1; done
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r2z_bench.log 2>&1

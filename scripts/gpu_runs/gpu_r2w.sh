cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_pytest.log 2>&1
timeout 300 python scripts/profile_epoch_host.py > gpurun_out/r2w_epoch_host.log 2>&1
timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2w_c5.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-secondary > gpurun_out/r2w_bench.log 2>&1
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2w_c3.log 2>&1

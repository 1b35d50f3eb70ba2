cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3o_pytest.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r3o_bench.log 2>&1
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3o_c3.log 2>&1

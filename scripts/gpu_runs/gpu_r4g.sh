cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r4g_pytest.log 2>&1; tail -1 gpurun_out/r4g_pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r4g_bench.log 2>&1

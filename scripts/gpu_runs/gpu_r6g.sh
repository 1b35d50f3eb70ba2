cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r6g_pytest.log 2>&1; tail -1 gpurun_out/r6g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6g_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r6g_smoke.log
timeout 900 python bench.py > gpurun_out/r6g_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/r6g_bench.log

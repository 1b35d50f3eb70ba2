cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4a_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r4a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r4a_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r4a_bench_ref.log 2>&1

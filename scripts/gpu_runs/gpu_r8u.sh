cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r8u_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r8u_pytest.log 2>&1; echo "pytest rc $? $(tail -1 gpurun_out/r8u_pytest.log)"
timeout 900 python bench.py > gpurun_out/r8u_bench.log 2>&1; echo "bench rc $?"

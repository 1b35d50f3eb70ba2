cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r8b_bench.log 2>&1; echo "rc $?" >> gpurun_out/r8b_bench.log

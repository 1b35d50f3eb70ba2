cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1b.log 2>&1

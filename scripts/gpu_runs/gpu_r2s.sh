cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_TRACE_REBUILD=3 timeout 600 python bench.py --workload c5 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2s_c5_trace.log 2>&1
TMD_TRACE_REBUILD=2 timeout 600 python bench.py --workload c5 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2s_c5_trace2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_c5_launches.csv python bench.py --workload c5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm > gpurun_out/r2s_ncu.log 2>&1

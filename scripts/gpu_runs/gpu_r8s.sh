cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r8s_launches_c5.csv python bench.py --workload c5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary --no-prewarm > gpurun_out/r8s_ncu.log 2>&1
echo "rc $?"

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
timeout 600 $CMD > gpurun_out/r8o_plain.log 2>&1; echo "plain rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r8o_launches.csv $CMD > gpurun_out/r8o_ncu_launch.log 2>&1
echo "launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_thread -s 1 -c 1 -f -o gpurun_out/r8o_build $CMD > gpurun_out/r8o_ncu_build.log 2>&1
echo "build rc $?"

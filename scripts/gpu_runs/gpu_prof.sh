cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1
echo "plain rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_lj -s 30 -c 1 -f -o gpurun_out/step_lj $CMD > gpurun_out/ncu_step.log 2>&1
echo "step rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_thread -s 1 -c 1 -f -o gpurun_out/build $CMD > gpurun_out/ncu_build.log 2>&1
echo "build rc $?"

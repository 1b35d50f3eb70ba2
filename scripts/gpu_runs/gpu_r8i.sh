cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
 timeout 900 python bench.py > gpurun_out/r8i_bench_$i.log 2>&1; echo "bench $i rc $?"
done
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r8i_launches.csv $CMD > gpurun_out/r8i_ncu_launch.log 2>&1
echo "launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_thread -s 1 -c 1 -f -o gpurun_out/r8i_build $CMD > gpurun_out/r8i_ncu_build.log 2>&1
echo "build rc $?"

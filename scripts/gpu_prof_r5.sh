# late-round-2 evidence: launch list of the bench command and full ncu captures of the
# step kernel (mid-epoch), the split list builder and the SD step kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches_bench20.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm --no-secondary > gpurun_out/r5_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 30 -c 1 -o gpurun_out/r5_k_step_lj python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm --no-secondary > gpurun_out/r5_ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_thread -s 1 -c 1 -o gpurun_out/r5_k_build python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm --no-secondary > gpurun_out/r5_ncu_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 30 -c 1 -o gpurun_out/r5_k_step_sd python bench.py --workload c5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm > gpurun_out/r5_ncu_sd.log 2>&1
ls -la gpurun_out/r5_*

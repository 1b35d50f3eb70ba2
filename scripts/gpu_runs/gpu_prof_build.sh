cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build_cells -s 1 -c 1 -o gpurun_out/r2_build_cells python bench.py --steps 25 --warmup 3 --no-cpu-baseline --no-e2e --no-prewarm > gpurun_out/r2_prof_build.log 2>&1

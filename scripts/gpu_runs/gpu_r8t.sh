cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r8t_summary.txt
for c in 2 1 3 4; do
 export TMD_NVCC_EXTRA="-DTMD_F32_CHUNK=$c"
 python -c "import sys; sys.path.insert(0,'paper_2009_07400_b200'); import build; build.build(force=True)" > gpurun_out/r8t_build_$c.log 2>&1 || { echo "build $c failed" >> gpurun_out/r8t_summary.txt; continue; }
 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_build --csv --log-file gpurun_out/r8t_build_$c.csv python bench.py --workload weak --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
 echo "chunk $c done" >> gpurun_out/r8t_summary.txt
done

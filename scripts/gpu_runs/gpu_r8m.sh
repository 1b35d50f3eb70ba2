cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r8m_summary.txt
for m in 1 8 9; do
 export TMD_NVCC_EXTRA="-DTMD_F32_MINB=$m"
 python -c "import sys; sys.path.insert(0,'paper_2009_07400_b200'); import build; build.build(force=True)" > gpurun_out/r8m_build_$m.log 2>&1 || { echo "build $m failed" >> gpurun_out/r8m_summary.txt; continue; }
 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_build --csv --log-file gpurun_out/r8m_build_$m.csv python bench.py --workload weak --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
 timeout 600 python bench.py --workload weak --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r8m_weak_$m.log 2>&1
 tail -1 gpurun_out/r8m_weak_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('weak minb=$m', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/r8m_summary.txt
done

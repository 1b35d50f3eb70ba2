cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r8k_summary.txt
for v in base lazy; do
 if [ $v = base ]; then export TMD_NVCC_EXTRA=""; else export TMD_NVCC_EXTRA="-DTMD_BUILD_LAZY_ID"; fi
 python -c "import sys; sys.path.insert(0,'paper_2009_07400_b200'); import build; build.build(force=True)" > gpurun_out/r8k_build_$v.log 2>&1 || { echo "build $v failed" >> gpurun_out/r8k_summary.txt; continue; }
 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_build --csv --log-file gpurun_out/r8k_build_$v.csv python bench.py --workload weak --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
 for i in 1 2; do
 timeout 600 python bench.py --workload weak --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r8k_weak_$v$i.log 2>&1
 tail -1 gpurun_out/r8k_weak_$v$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('weak $v', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/r8k_summary.txt
 done
done
export TMD_NVCC_EXTRA="-DTMD_BUILD_LAZY_ID"
python -c "import sys; sys.path.insert(0,'paper_2009_07400_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r8k_pytest_lazy.log 2>&1; tail -1 gpurun_out/r8k_pytest_lazy.log >> gpurun_out/r8k_summary.txt

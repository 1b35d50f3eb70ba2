cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r8x_summary.txt
for b in 1 0; do
 export TMD_NVCC_EXTRA="-DTMD_STEP_BALANCE=$b"
 python -c "import sys; sys.path.insert(0,'paper_2009_07400_b200'); import build; build.build(force=True)" > gpurun_out/r8x_build_$b.log 2>&1 || { echo "build $b failed" >> gpurun_out/r8x_summary.txt; continue; }
 for i in 1 2; do
 for w in weak c5; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r8x_${w}_$b$i.log 2>&1
  tail -1 gpurun_out/r8x_${w}_$b$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w balance=$b', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['kernel_ms_median'],4))" >> gpurun_out/r8x_summary.txt
 done
 done
done
export TMD_NVCC_EXTRA="-DTMD_STEP_BALANCE=1"
python -c "import sys; sys.path.insert(0,'paper_2009_07400_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r8x_pytest.log 2>&1; tail -1 gpurun_out/r8x_pytest.log >> gpurun_out/r8x_summary.txt

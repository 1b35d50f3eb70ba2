cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r8c_pytest.log 2>&1; tail -1 gpurun_out/r8c_pytest.log
rm -f gpurun_out/r8c_summary.txt
for i in 1 2; do
 for g in 1 0; do
  for w in weak c5 c3; do
  TMD_EPOCH_GRAPH=$g timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r8c_${w}_$g$i.log 2>&1
  tail -1 gpurun_out/r8c_${w}_$g$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w graph=$g', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/r8c_summary.txt
  done
 done
done

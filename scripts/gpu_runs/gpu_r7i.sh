cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r7i_pytest.log 2>&1; tail -1 gpurun_out/r7i_pytest.log
rm -f gpurun_out/r7i_summary.txt
for i in 1 2; do
  for w in weak c5; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r7i_${w}_$i.log 2>&1
  tail -1 gpurun_out/r7i_${w}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/r7i_summary.txt
  done
done

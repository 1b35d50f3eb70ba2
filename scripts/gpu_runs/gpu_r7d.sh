cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r7d_summary.txt
for i in 1 2; do
 for v in 1 0; do
  for w in weak c5; do
  TMD_PREPARE_EARLY=$v timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r7d_${w}_$v$i.log 2>&1
  tail -1 gpurun_out/r7d_${w}_$v$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w early=$v', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/r7d_summary.txt
  done
 done
done

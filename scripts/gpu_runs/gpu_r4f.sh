cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r4f_summary.txt
for c in 0.5 0.4 0.3 0.5 0.4 0.3; do
  TMD_MARGIN_CAP=$c timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r4f_$c.log 2>&1
  tail -1 gpurun_out/r4f_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['kernel_ms_median'],4))" >> gpurun_out/r4f_summary.txt
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r8p_summary.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r8p_pytest.log 2>&1; tail -1 gpurun_out/r8p_pytest.log >> gpurun_out/r8p_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_build|k_cell_positions" --csv --log-file gpurun_out/r8p_build.csv python bench.py --workload weak --steps 40 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
for i in 1 2; do
 for w in weak c5 c3; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r8p_${w}_$i.log 2>&1
  tail -1 gpurun_out/r8p_${w}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/r8p_summary.txt
 done
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for o in cell brick cell brick; do
TMD_ORDER=$o TMD_TRACE_REBUILD=3 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench1_$o.log 2>&1
tail -1 gpurun_out/bench1_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', round(d['value']/1e9,3), round(d['roofline']['kernel_ms'],4), [r['lists'] for r in d['outliers']['rebuild_device_ms']])"
done

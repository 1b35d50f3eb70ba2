cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 4 8 0 8 4; do
TMD_BUILD_CHUNK=$v TMD_TRACE_REBUILD=3 timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench1_c$v.log 2>&1
tail -1 gpurun_out/bench1_c$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk', $v, round(d['value']/1e9,3), [r['lists'] for r in d['outliers']['rebuild_device_ms']])"
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_LIST_SHELL=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lj80 or lj32 or fused or production" > gpurun_out/r6b_pytest_s3.log 2>&1; tail -1 gpurun_out/r6b_pytest_s3.log
rm -f gpurun_out/r6b_summary.txt
for sh in 2 3 2 3; do
  TMD_LIST_SHELL=$sh timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r6b_$sh.log 2>&1
  tail -1 gpurun_out/r6b_$sh.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$sh', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['kernel_ms_median'],4))" >> gpurun_out/r6b_summary.txt
done
for sh in 2 3; do TMD_LIST_SHELL=$sh timeout 300 python scripts/profile_rebuild.py 80 2>&1 | grep "k_build" >> gpurun_out/r6b_build_$sh.log; done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 1 6 8; do
  TMD_STEP_MINB=$m timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_minb$m.log 2>&1
done
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 300 python scripts/profile_rebuild.py --cells 80 > gpurun_out/rebuild_weak.log 2>&1
timeout 600 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_weak.log 2>&1
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_weak.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_weak.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 300 python scripts/profile_rebuild.py --cells 32 > gpurun_out/rebuild_c2.log 2>&1
timeout 300 python scripts/profile_rebuild.py --cells 80 > gpurun_out/rebuild_weak.log 2>&1
timeout 600 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_weak.log 2>&1
CMD2="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > gpurun_out/plain_weak.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_lj -s 6 -c 1 -o gpurun_out/prof_step_weak3 $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done

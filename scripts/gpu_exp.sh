cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python scripts/profile_epoch.py --cells 80 > gpurun_out/epoch_weak.log 2>&1
timeout 600 python scripts/experiments/exp_force.py 80 > gpurun_out/exp_force.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_weak_$i.log 2>&1; done
CMD="python scripts/profile_epoch.py --cells 80 --steps 45"
timeout 300 $CMD > gpurun_out/epoch_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_epoch.csv $CMD > gpurun_out/ncu_epoch.log 2>&1
echo done

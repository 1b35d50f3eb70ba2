cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_weak.log 2>&1
timeout 600 python bench.py --workload c2 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
if [ "$NG" -ge 2 ]; then
  timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/mgpu_$NG.log 2>&1
  echo "mgpu exit $?" >> gpurun_out/mgpu_$NG.log
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 100 --warmup 5 > gpurun_out/bench_weak_n$NG.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench_weak_n$NG.log
fi
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_weak.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_weak.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 300 $CMD > gpurun_out/plain_weak2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_lj -s 8 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_step.log 2>&1
timeout 300 $CMD > gpurun_out/plain_weak3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_build -s 1 -c 1 -o gpurun_out/prof_build $CMD > gpurun_out/ncu_build.log 2>&1
echo done

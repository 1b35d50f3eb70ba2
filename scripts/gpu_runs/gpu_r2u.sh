cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/profile_epoch_host.py > gpurun_out/r2u_epoch_host.log 2>&1
timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2u_c5.log 2>&1

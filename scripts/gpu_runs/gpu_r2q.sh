cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2q_ref.log 2>&1
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2q_bench.log 2>&1
timeout 600 python scripts/exp_half.py 80 > gpurun_out/r2q_half.log 2>&1
nproc > gpurun_out/r2q_nproc.txt; free -g >> gpurun_out/r2q_nproc.txt

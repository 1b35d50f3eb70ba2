cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/diag_c5_secondary.py > gpurun_out/r3p_c5sec.log 2>&1
timeout 300 python scripts/diag_c5_secondary.py big > gpurun_out/r3p_c5sec_big.log 2>&1

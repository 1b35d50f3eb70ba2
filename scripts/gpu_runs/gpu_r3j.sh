cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_BUILD_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or lists or fused or lj80 or lj32" > gpurun_out/r3j_pytest_v1.log 2>&1
for v in 0 1; do TMD_BUILD_VARIANT=$v timeout 300 python scripts/profile_rebuild.py 80 > gpurun_out/r3j_rebuild_v$v.log 2>&1; done
for v in 0 1; do TMD_BUILD_VARIANT=$v timeout 300 python scripts/profile_rebuild.py 80 > gpurun_out/r3j_rebuild2_v$v.log 2>&1; done

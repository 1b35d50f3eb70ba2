cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_BUILD_VARIANT=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or lists or fused or lj80 or lj32" > gpurun_out/r3l_pytest_v2.log 2>&1
for v in 1 2 1 2; do TMD_BUILD_VARIANT=$v timeout 300 python scripts/profile_rebuild.py 80 2>&1 | grep "k_build" >> gpurun_out/r3l_build_v$v.log; done

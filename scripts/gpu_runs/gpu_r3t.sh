cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_BUILD_AOS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or lists or fused or lj80 or lj32" > gpurun_out/r3t_pytest_aos.log 2>&1
for v in 0 1 0 1; do TMD_BUILD_AOS=$v timeout 300 python scripts/profile_rebuild.py 80 2>&1 | grep "k_build\|k_pack_cp4" >> gpurun_out/r3t_build_aos$v.log; done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r3n_build_v*.log
for v in 4 5 6 4 5 6; do TMD_BUILD_VARIANT=$v timeout 300 python scripts/profile_rebuild.py 80 2>&1 | grep "k_build" >> gpurun_out/r3n_build_v$v.log; done

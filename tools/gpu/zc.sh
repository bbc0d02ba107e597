cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/micro/zerocopy > gpurun_out/zerocopy.log 2>&1; echo "rc=$?" >> gpurun_out/zerocopy.log

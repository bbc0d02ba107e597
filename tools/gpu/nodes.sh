cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/node_sizes.py 131072 0 > gpurun_out/nodes_c3.log 2>&1
timeout 900 python tools/node_sizes.py 32768 0 > gpurun_out/nodes_c2.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --kv-offload --steps 48 --warmup 5 --no-cpu-baseline > gpurun_out/b_c2_off.log 2>&1; echo "rc=$?" >> gpurun_out/b_c2_off.log
timeout 1500 python bench.py --kv-offload --ctx 131072 --steps 32 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3_off.log 2>&1; echo "rc=$?" >> gpurun_out/b_c3_off.log

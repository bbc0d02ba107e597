cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider --timeout 600 -rf -k "offload" > gpurun_out/off_tests.log 2>&1; echo "rc=$?" >> gpurun_out/off_tests.log
timeout 1500 python bench.py --kv-offload --ctx 131072 --steps 32 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3_off.log 2>&1; echo "rc=$?" >> gpurun_out/b_c3_off.log

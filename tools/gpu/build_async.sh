cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/async_tests.log 2>&1; echo "rc=$?" >> gpurun_out/async_tests.log
for g in 1 4 8; do timeout 1200 python tools/llama_prefill.py 32768 64 $g; done > gpurun_out/llama_groups.log 2>&1
timeout 600 python tools/time_prefill.py > gpurun_out/prefill_c2.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for g in 1 4 10; do timeout 1200 python tools/llama_prefill.py 32768 64 $g; done > gpurun_out/llama_groups.log 2>&1
timeout 600 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider --timeout 600 -rf -k "layer_streaming" >> gpurun_out/llama_groups.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider --timeout 600 -rf -k "layer_streaming or llama" > gpurun_out/llama_tests.log 2>&1; echo "rc=$?" >> gpurun_out/llama_tests.log
timeout 900 python tools/llama_prefill.py 8192 32 > gpurun_out/llama_8k.log 2>&1; echo "rc=$?" >> gpurun_out/llama_8k.log
timeout 1200 python tools/llama_prefill.py 32768 64 > gpurun_out/llama_32k.log 2>&1; echo "rc=$?" >> gpurun_out/llama_32k.log

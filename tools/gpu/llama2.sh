cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/llama_prefill.py 32768 64 > gpurun_out/llama_32k_prio.log 2>&1; echo "rc=$?" >> gpurun_out/llama_32k_prio.log
timeout 900 python tools/llama_prefill.py 8192 32 > gpurun_out/llama_8k_prio.log 2>&1; echo "rc=$?" >> gpurun_out/llama_8k_prio.log

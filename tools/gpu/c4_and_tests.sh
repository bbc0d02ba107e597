cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --seqs-per-gpu 8 --steps 32 --warmup 5 --no-cpu-baseline > gpurun_out/b_c4s8.log 2>&1; echo "rc=$?" >> gpurun_out/b_c4s8.log
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_engine_ref_api.py tests/test_gpu_engine_api.py tests/test_gpu_forest.py -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/gputest2.log 2>&1; echo "rc=$?" >> gpurun_out/gputest2.log
timeout 600 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/b_default2.log 2>&1; echo "rc=$?" >> gpurun_out/b_default2.log

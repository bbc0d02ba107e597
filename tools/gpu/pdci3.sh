cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dci_api.py tests/test_gpu_forest.py tests/test_gpu_acceptance.py tests/test_gpu_large.py tests/test_gpu_engine.py -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pdci_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdci_tests.log
ICB_PROF=1 timeout 600 python tools/time_rotation.py 32768 > gpurun_out/rot_c2.log 2>&1
ICB_PROF=1 timeout 900 python tools/time_rotation.py 131072 > gpurun_out/rot_c3.log 2>&1
timeout 900 python bench.py --ctx 131072 --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3.log 2>&1; echo "rc=$?" >> gpurun_out/b_c3.log
timeout 900 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/b_c2.log 2>&1; echo "rc=$?" >> gpurun_out/b_c2.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_forest.py -q -p no:cacheprovider --timeout 300 -rf -k "dense" > gpurun_out/dense_test.log 2>&1; echo "rc=$?" >> gpurun_out/dense_test.log
timeout 300 python tools/bench_dense.py > gpurun_out/dense_bench.log 2>&1; echo "rc=$?" >> gpurun_out/dense_bench.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
  for mode in order none; do
    if [ $mode = none ]; then export ICB_NO_ORDER=1; else unset ICB_NO_ORDER; fi
    printf "%-8s " $mode
    python bench.py --steps 128 --warmup 8 --no-cpu-baseline 2>&1 | tail -1 | python tools/summ.py | cut -c1-110
  done
done > gpurun_out/ab_order.log 2>&1
unset ICB_NO_ORDER
for mode in order none; do
  if [ $mode = none ]; then export ICB_NO_ORDER=1; else unset ICB_NO_ORDER; fi
  printf "%-8s " $mode
  python bench.py --ctx 131072 --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | tail -1 | python tools/summ.py | cut -c1-110
done > gpurun_out/ab_order_c3.log 2>&1
unset ICB_NO_ORDER
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_large.py -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/order_tests.log 2>&1; echo "rc=$?" >> gpurun_out/order_tests.log

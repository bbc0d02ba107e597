cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/gputest1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest1.log
timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench1.log

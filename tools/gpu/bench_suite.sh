cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b_default.log 2>&1; echo "rc=$?" >> gpurun_out/b_default.log
timeout 600 python bench.py --check > gpurun_out/b_check.log 2>&1; echo "rc=$?" >> gpurun_out/b_check.log
timeout 600 python bench.py --kv fp32 --steps 64 --warmup 8 --no-cpu-baseline > gpurun_out/b_fp32.log 2>&1; echo "rc=$?" >> gpurun_out/b_fp32.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b_ref.log 2>&1; echo "rc=$?" >> gpurun_out/b_ref.log
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt

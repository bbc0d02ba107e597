cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/b_c2.log 2>&1; echo "rc=$?" >> gpurun_out/b_c2.log
timeout 900 python bench.py --ctx 131072 --steps 32 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3.log 2>&1; echo "rc=$?" >> gpurun_out/b_c3.log
timeout 300 python tools/prof_query.py 32768 bf16 12 > gpurun_out/pq_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"query_kernel|attn_kernel|dense_flash|insert_kernel|append|dense_append|rotate" -c 120 --csv --log-file gpurun_out/launches_c2.csv python tools/prof_query.py 32768 bf16 12 > gpurun_out/ncu_l.log 2>&1
timeout 300 python tools/prof_query.py 131072 bf16 6 > gpurun_out/pq_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_flash -s 2 -c 1 -o gpurun_out/prof_flash_c3 -f python tools/prof_query.py 131072 bf16 6 > gpurun_out/ncu_f3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_flash -s 2 -c 1 -o gpurun_out/prof_flash_c2 -f python tools/prof_query.py 32768 bf16 12 > gpurun_out/ncu_f2.log 2>&1
echo finished >> gpurun_out/ncu_f2.log

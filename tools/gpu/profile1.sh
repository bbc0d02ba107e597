cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_phases.py > gpurun_out/phases.log 2>&1
timeout 900 python bench.py --seqs-per-gpu 8 --steps 32 --warmup 5 --no-cpu-baseline > gpurun_out/b_c4s8.log 2>&1; echo "rc=$?" >> gpurun_out/b_c4s8.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/b_c4s8.log
timeout 300 python tools/prof_query.py > gpurun_out/pq_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_kernel -s 6 -c 1 -o gpurun_out/prof_query -f python tools/prof_query.py > gpurun_out/ncu_q.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 6 -c 1 -o gpurun_out/prof_dense -f python tools/prof_query.py > gpurun_out/ncu_d.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches.csv python tools/prof_query.py > gpurun_out/ncu_l.log 2>&1
echo finished >> gpurun_out/ncu_l.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for cfg in "32768 bf16 c2" "131072 bf16 c3" "32768 fp32 c2fp32"; do
  set -- $cfg
  timeout 600 python tools/prof_query.py $1 $2 > $O/pq_$3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_kernel -s 6 -c 1 -o /tmp/prof_query_$3 -f python tools/prof_query.py $1 $2 > $O/ncu_$3.log 2>&1 && \
  python tools/ncu_summary.py /tmp/prof_query_$3.ncu-rep query_kernel $O/r02_query_kernel_$3_ncu_summary.json > /dev/null 2>&1; \
  python tools/ncu_lines.py /tmp/prof_query_$3.ncu-rep 40 > $O/lines_$3.txt 2>&1; \
  python tools/ncu_traffic.py /tmp/prof_query_$3.ncu-rep ctx$1_$2_s1 "ncu --set full, query_kernel (tools/prof_query.py $1 $2), profiles/r02_query_kernel_$3_ncu_summary.json" >> $O/traffic.log 2>&1
done
cp profiles/search_traffic.json $O/search_traffic.json
timeout 900 python bench.py > $O/b_default.log 2>&1; echo "rc=$?" >> $O/b_default.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/b_k20.log 2>&1; echo "rc=$?" >> $O/b_k20.log
timeout 900 python bench.py --ctx 131072 --steps 64 --warmup 5 --no-cpu-baseline > $O/b_c3.log 2>&1; echo "rc=$?" >> $O/b_c3.log
timeout 900 python bench.py --kv fp32 --steps 64 --warmup 8 --no-cpu-baseline > $O/b_fp32.log 2>&1; echo "rc=$?" >> $O/b_fp32.log
timeout 900 python bench.py --seqs-per-gpu 8 --steps 32 --warmup 5 --no-cpu-baseline > $O/b_c4s8.log 2>&1; echo "rc=$?" >> $O/b_c4s8.log
timeout 900 python bench.py --kv-offload --steps 32 --warmup 5 --no-cpu-baseline > $O/b_c2_off.log 2>&1; echo "rc=$?" >> $O/b_c2_off.log
timeout 900 python bench.py --kv-offload --ctx 131072 --steps 32 --warmup 5 --no-cpu-baseline > $O/b_c3_off.log 2>&1; echo "rc=$?" >> $O/b_c3_off.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/b_ref.log 2>&1; echo "rc=$?" >> $O/b_ref.log
timeout 600 python bench.py --check > $O/b_check.log 2>&1; echo "rc=$?" >> $O/b_check.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "rc=$?" >> $O/ncu_launches.log
echo done > $O/done

# refreshed final evidence after the mapped-report / double-staging change
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/final2_bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/final2_bench_c1.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final2_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/final2_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final2_launches_c1.csv python bench.py --steps 30 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/final2_ncu_launches.log 2>&1; echo "ncu rc=$?" >> gpurun_out/final2_ncu_launches.log
tail -2 gpurun_out/smoke.log
grep '^{' gpurun_out/final2_bench_c1.log | cut -c1-400
tail -1 gpurun_out/final2_ncu_launches.log

# Final round-1 evidence: default bench, C2, llama3-8b, ncu launch list of the default command,
# ncu --set full of the packed tensor-core kernel (short and long items)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_c1.log
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline > gpurun_out/final_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_c2.log
timeout 900 python bench.py --shape llama3-8b --no-cpu-baseline > gpurun_out/final_bench_llama.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_llama.log
timeout 900 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-chunks 32 > gpurun_out/final_bench_e2e32.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_e2e32.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_launches_c1.csv python bench.py --steps 30 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/final_ncu_launches.log 2>&1; echo "ncu rc=$?" >> gpurun_out/final_ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/final_attn_tc_short python tools/attn_sweep.py --case "tc short" --steps 3 > gpurun_out/final_ncu_tc_short.log 2>&1; echo "rc=$?" >> gpurun_out/final_ncu_tc_short.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/final_attn_tc_gqa python tools/attn_sweep.py --case "llama3-8b gqa tc" --steps 3 > gpurun_out/final_ncu_tc.log 2>&1; echo "rc=$?" >> gpurun_out/final_ncu_tc.log
for f in final_bench_c1 final_bench_c2 final_bench_llama final_bench_e2e32; do tail -1 gpurun_out/$f.log; grep '^{' gpurun_out/$f.log | cut -c1-300; done

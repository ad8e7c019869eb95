cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/attn_tc_gqa2 python tools/attn_sweep.py --case "llama3-8b gqa tc" --steps 3 > gpurun_out/ncu_tc.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_tc.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_llama_tc_fused.csv python bench.py --shape llama3-8b --steps 30 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/ncu_llama.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_llama.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1.log
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 30 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tma -s 60 -c 1 -o gpurun_out/attn_fused python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --arena-gb 80 > gpurun_out/ncu_fused.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_fused.log

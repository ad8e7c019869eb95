cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c1.log
timeout 600 python bench.py --config c2 --p 0.1 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_attn|k_move" -c 40 --csv --log-file gpurun_out/traffic_c2.csv python bench.py --config c2 --p 0.1 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_traffic.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_traffic.log

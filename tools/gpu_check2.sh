cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --arena-gb 40 > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 3 -c 1 -o gpurun_out/attn python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --arena-gb 40 > gpurun_out/ncu_attn.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/ncu_attn.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_move -s 0 -c 1 -o gpurun_out/move python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --arena-gb 40 > gpurun_out/ncu_move.log 2>&1; echo "ncu3 rc=$?" >> gpurun_out/ncu_move.log
timeout 600 python bench.py --config c2 --p 0.1 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log

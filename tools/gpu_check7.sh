cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_pass.log 2>&1
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline --no-e2e --compact fused > gpurun_out/bench_c2_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tma -s 40 -c 1 -o gpurun_out/attn_fused python bench.py --config c2 --p 0.1 --steps 45 --warmup 3 --no-e2e --no-cpu-baseline --arena-gb 40 --compact fused > gpurun_out/ncu_fused.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_fused.log

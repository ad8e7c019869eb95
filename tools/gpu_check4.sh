cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in tma regs; do
timeout 600 python bench.py --attn $v --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_$v.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c1_$v.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tma -s 3 -c 1 -o gpurun_out/attn_tma python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --arena-gb 40 > gpurun_out/ncu_attn_tma.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_attn_tma.log

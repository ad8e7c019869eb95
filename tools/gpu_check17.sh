cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --shape llama3-8b --requests 32768 --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/bench_llama_tc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama_tc.log
timeout 900 python bench.py --shape llama3-8b --requests 32768 --no-cpu-baseline --no-e2e --steps 100 --attn tma > gpurun_out/bench_llama_tma.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama_tma.log
timeout 900 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1.log

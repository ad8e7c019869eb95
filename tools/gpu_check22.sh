cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "tensor_cores or randomized" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 python bench.py --shape llama3-8b --attn tc --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_llama_tc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama_tc.log
timeout 600 python bench.py --shape llama3-8b --attn tc --config c2 --p 0.1 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_llama_tc_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama_tc_c2.log

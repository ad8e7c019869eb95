cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores or randomized" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python tools/attn_sweep.py --case "tc" > gpurun_out/attn_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/attn_sweep.log
timeout 600 python bench.py --shape llama3-8b --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_llama_tc.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama_tc.log

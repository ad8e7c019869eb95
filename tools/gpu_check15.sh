cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/attn_sweep.py > gpurun_out/attn_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/attn_sweep.log
timeout 900 python bench.py --shape llama3-8b --requests 32768 --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/bench_llama.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama.log

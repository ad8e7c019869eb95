# TC: 8-row load granularity; parity + A/B against HEAD (packed, 16-row groups)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores or host_fed or grouped or abi_error" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -2 gpurun_out/pytest_tc.log
echo "== new"; timeout 200 python tools/attn_sweep.py --case "tc" 2>&1 | grep case
echo "== head"; timeout 200 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case
timeout 600 python bench.py --shape llama3-8b --no-cpu-baseline --no-e2e > gpurun_out/bench_llama.log 2>&1
grep '^{' gpurun_out/bench_llama.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('llama bench', d['value'], d['ms_per_step'], d['roofline']['frac'])"

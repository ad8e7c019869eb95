# tensor-core kernel appends the new row itself (no k_append) and waits on host-fed ready words
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores or host_fed or grouped or randomized or abi_error" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -3 gpurun_out/pytest_tc.log
echo "== new"; timeout 200 python tools/attn_sweep.py --case "tc" 2>&1 | grep case | cut -c1-60,150-
echo "== head"; timeout 200 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case | cut -c1-60,150-
timeout 900 python bench.py --shape llama3-8b --no-cpu-baseline > gpurun_out/bench_llama.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama.log
grep '^{' gpurun_out/bench_llama.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('llama', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'])"

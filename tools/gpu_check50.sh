# ping-pong softmax groups in the tensor-core kernel: parity first (short timeout), then A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -3 gpurun_out/pytest_tc.log
grep -q "pytest rc=0" gpurun_out/pytest_tc.log || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grouped or host_fed or randomized" > gpurun_out/pytest_tc2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc2.log
tail -2 gpurun_out/pytest_tc2.log
echo "== new"; timeout 300 python tools/attn_sweep.py --case "tc" --custom "len16 tc:32,32,8,128,8192,15,2" --custom "len100 tc:32,32,8,128,4096,99,2" 2>&1 | grep case | cut -c1-60,150-
echo "== head"; timeout 300 python tools/attn_sweep.py --case "tc" --custom "len16 tc:32,32,8,128,8192,15,2" --custom "len100 tc:32,32,8,128,4096,99,2" --lib tools/ab/libs3_head.so 2>&1 | grep case | cut -c1-60,150-
timeout 600 python bench.py --shape llama3-8b --no-cpu-baseline --no-e2e > gpurun_out/bench_llama.log 2>&1
grep '^{' gpurun_out/bench_llama.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('llama', d['value'], d['ms_per_step'], d['roofline']['frac'])"

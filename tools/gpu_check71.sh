# hybrid: full tiles block-major (2-D boxes), partial tiles 4-D boxes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -2 gpurun_out/pytest_tc.log
grep -q "pytest rc=0" gpurun_out/pytest_tc.log || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grouped or host_fed or layer_group or double_buffered or randomized" > gpurun_out/pytest_tc2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc2.log
tail -2 gpurun_out/pytest_tc2.log
echo "== new"; timeout 300 python tools/attn_sweep.py --case "tc" 2>&1 | grep case | cut -c1-40,150-
echo "== head"; timeout 300 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case | cut -c1-40,150-
timeout 900 python bench.py --shape llama3-8b --no-cpu-baseline --no-e2e > gpurun_out/bench_llama.log 2>&1
grep '^{' gpurun_out/bench_llama.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('llama', round(d['value']), round(d['roofline']['frac'],3))"

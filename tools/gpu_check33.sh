# TC kernel: double p_full (two-phase hazard) + PACK template; hang hunt + parity + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
echo "== new mqa $i"; timeout 90 python tools/attn_sweep.py --case "mqa H=16 D=128 tc" 2>&1 | grep case
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores or host_fed" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -2 gpurun_out/pytest_tc.log
echo "== new"; timeout 200 python tools/attn_sweep.py --case "tc" 2>&1 | grep case
echo "== head"; timeout 200 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case
timeout 600 python bench.py --shape llama3-8b --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_llama.log 2>&1
grep '^{' gpurun_out/bench_llama.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('llama bench', d['value'], d['ms_per_step'], d['roofline']['frac'])"

# TC kernel: short KV heads packed two per tile (block-diagonal scores); parity + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S3_TC_PACK=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -3 gpurun_out/pytest_tc.log
for pk in 2; do
S3_TC_PACK=$pk timeout 600 python tools/attn_sweep.py --case "tc" > gpurun_out/attn_sweep_pack$pk.log 2>&1
echo "pack=$pk"; cat gpurun_out/attn_sweep_pack$pk.log | grep case
S3_TC_PACK=$pk timeout 600 python bench.py --shape llama3-8b --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_llama_pack$pk.log 2>&1
python -c "
import json
for l in open('gpurun_out/bench_llama_pack$pk.log'):
    if l.startswith('{'):
        d=json.loads(l); print('pack=$pk', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'])
"; tail -2 gpurun_out/bench_llama_pack$pk.log | grep -v '^{'
done

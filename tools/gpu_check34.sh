# o_done waited every tile (synccheck); k_synth row-blocked; HBM ceiling probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 tools/hbm_probe/hbm_probe > gpurun_out/hbm_probe.json 2>&1; cat gpurun_out/hbm_probe.json
echo "== new"; timeout 200 python tools/attn_sweep.py --case "tc" 2>&1 | grep case
echo "== head"; timeout 200 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case
timeout 1200 compute-sanitizer --tool synccheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores and (4-2-7 or 8-2-64)" > gpurun_out/sanitize3_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize3_synccheck.log
tail -4 gpurun_out/sanitize3_synccheck.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_k30.log 2>&1
grep '^{' gpurun_out/bench_k30.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('gptj k30', d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'], d['roofline'].get('context'))"

# final checks after the N=32 PV / 3-D q changes: sanitizers on the tensor-core tests, full suite, LLaMA bench, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores and (4-2-7 or 8-2-64 or 16-1-128) or host_fed_decode_step and 2-0-16" > gpurun_out/sanitize5_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize5_$tool.log
  tail -3 gpurun_out/sanitize5_$tool.log
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --shape llama3-8b --no-cpu-baseline > gpurun_out/final_bench_llama.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_llama.log
grep '^{' gpurun_out/final_bench_llama.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print('llama', round(d['value']), round(r['achieved']), round(r['frac'],3), r['context']['frac_of_read_ceiling'], round(d['ms_per_step'],2), round(d['e2e']['value']))"
timeout 300 python tools/attn_sweep.py --case "tc" > gpurun_out/final_sweep_tc.log 2>&1; grep case gpurun_out/final_sweep_tc.log | cut -c1-50,150-
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/final_attn_tc_short2 python tools/attn_sweep.py --case "tc short" --steps 3 > gpurun_out/final_ncu_tc_short2.log 2>&1; echo "rc=$?" >> gpurun_out/final_ncu_tc_short2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/final_attn_tc_gqa2 python tools/attn_sweep.py --case "llama3-8b gqa tc" --steps 3 > gpurun_out/final_ncu_tc2.log 2>&1; echo "rc=$?" >> gpurun_out/final_ncu_tc2.log

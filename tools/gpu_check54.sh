# full GPU suite + LLaMA bench after the N = 32 PV MMA
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --shape llama3-8b --no-cpu-baseline > gpurun_out/bench_llama.log 2>&1; echo "rc=$?" >> gpurun_out/bench_llama.log
grep '^{' gpurun_out/bench_llama.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print('llama', round(d['value']), round(r['achieved']), round(r['frac'],3), r['context']['frac_of_read_ceiling'], round(d['ms_per_step'],2), round(d['e2e']['value']))"
timeout 300 python tools/attn_sweep.py --case "len" --custom "len16:32,32,8,128,8192,15,2" --custom "len32:32,32,8,128,8192,31,2" --custom "len100:32,32,8,128,4096,99,2" --custom "len250:32,32,8,128,2048,249,2" 2>&1 | grep case | cut -c1-30,150-

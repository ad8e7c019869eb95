# final lines after the generator speedups
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/final3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final3_pytest.log
tail -2 gpurun_out/final3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final3_smoke.log; tail -1 gpurun_out/final3_smoke.log
timeout 900 python bench.py > gpurun_out/final3_c1.log 2>&1
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline > gpurun_out/final3_c2.log 2>&1
timeout 900 python bench.py --shape llama3-8b --no-cpu-baseline > gpurun_out/final3_llama.log 2>&1
for f in final3_c1 final3_c2 final3_llama; do grep '^{' gpurun_out/$f.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', round(d['value']), round(d['ms_per_step'],2), round(r['achieved']), round(r['frac'],3), r['context']['frac_of_read_ceiling'], round(d['e2e']['value']), d['evict_compact']['evicted'], d['clocks']['sm_mhz'], d['cpu_baseline'] and round(d['cpu_baseline']['value'],1))"; done

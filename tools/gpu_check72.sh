# default bench after the guard-row change (arena R + 8 rows)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f5_c1.log 2>&1; echo "rc=$?" >> gpurun_out/f5_c1.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f5_ref.log 2>&1
grep '^{' gpurun_out/f5_c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('c1', round(d['value']), round(d['ms_per_step'],2), round(r['achieved']), round(r['frac'],3), r['context']['frac_of_read_ceiling'], round(d['e2e']['value']), d['clocks'], d['gpu_launches'], round(d['cpu_baseline']['value'],1))"
tail -n 1 gpurun_out/f5_c1.log
grep -c '^{' gpurun_out/f5_ref.log

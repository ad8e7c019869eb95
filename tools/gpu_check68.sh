# whole-run C1: 8192 requests stepped to (near) completion in the timed region
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 1400 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c1_wholerun.log 2>&1; echo "rc=$?" >> gpurun_out/c1_wholerun.log
grep '^{' gpurun_out/c1_wholerun.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(round(d['value']), d['tokens'], d['finished'], d['admitted'], round(d['ms_per_step'],2), round(r['frac'],3), d['config']['mean_batch'], d['latency_split']['penalty_plus_overhead_share'])"

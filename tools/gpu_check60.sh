# round-end rehearsal: what the driver runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/rehearsal_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rehearsal_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rehearsal_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rehearsal_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/rehearsal_ref.log 2>&1; echo "rc=$?" >> gpurun_out/rehearsal_ref.log
timeout 900 python bench.py > gpurun_out/rehearsal_bench.log 2>&1; echo "rc=$?" >> gpurun_out/rehearsal_bench.log
tail -2 gpurun_out/rehearsal_pytest.log gpurun_out/rehearsal_smoke.log
grep '^{' gpurun_out/rehearsal_ref.log | cut -c1-160
grep '^{' gpurun_out/rehearsal_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],2), round(r['frac'],3), r['context']['frac_of_read_ceiling'], round(d['e2e']['value']), d['clocks'], d['gpu_launches'])"

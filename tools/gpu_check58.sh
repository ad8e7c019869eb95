# e2e pipeline depth sweep (default C1 window of the e2e leg)
cd $GRAFT_REPO_ROOT
for c in 8 12 16 24; do
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-chunks $c > gpurun_out/e2e_$c.log 2>&1
grep '^{' gpurun_out/e2e_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']; print($c, round(e['value']), e['ms_per_step'], e['pcie_gbs'])"
done

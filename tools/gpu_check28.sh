cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 16 64; do
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-chunks $c > gpurun_out/bench_e2e_$c.log 2>&1
python -c "
import json
for l in open('gpurun_out/bench_e2e_$c.log'):
    if l.startswith('{'):
        d=json.loads(l); print($c, d['value'], d['phases_ms_per_step'], d['e2e'])
"; tail -1 gpurun_out/bench_e2e_$c.log; done

# host-fed decode step (s3_decode_step_host): parity + e2e pipeline depth sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_fed" > gpurun_out/pytest_hostfed.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hostfed.log
for c in 16 4 1; do
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-chunks $c > gpurun_out/bench_e2e_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_e2e_$c.log
done
tail -3 gpurun_out/pytest_hostfed.log
for c in 16 4 1; do python -c "
import json,sys
for l in open('gpurun_out/bench_e2e_$c.log'):
    if l.startswith('{'):
        d=json.loads(l); print($c, d['value'], d['e2e'])
"; tail -2 gpurun_out/bench_e2e_$c.log; done

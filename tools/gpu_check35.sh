# host-fed step with device out + per-chunk D2H (stream waits on kernel counters)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_fed" > gpurun_out/pytest_hostfed.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hostfed.log
tail -3 gpurun_out/pytest_hostfed.log
for mode in "" "--e2e-mapped-out"; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline $mode > gpurun_out/bench_e2e.log 2>&1
grep '^{' gpurun_out/bench_e2e.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$mode', d['value'], d['e2e'])"
tail -2 gpurun_out/bench_e2e.log | grep -v '^{'
done

# double-buffered eviction staging: full GPU suite + C2 overlap evidence
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for p in 0.1 0.2; do
timeout 900 python bench.py --config c2 --p $p --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_$p.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2_$p.log
grep '^{' gpurun_out/bench_c2_$p.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$p', d['value'], d['ms_per_step'], d['evict_compact']['evicted'], d['pcie'])"
done

# report written by k_prep into mapped pinned memory (no CE queueing behind eviction D2H)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for p in 0.1 0.2; do
timeout 900 python bench.py --config c2 --p $p --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_$p.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2_$p.log
grep '^{' gpurun_out/bench_c2_$p.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$p', d['value'], d['ms_per_step'], d['evict_compact']['evicted'], d['pcie']['evict_d2h_ms'], d['pcie']['evict_d2h_overlapped_with_attention_frac'])"
done
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1
grep '^{' gpurun_out/bench_c1.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c1', d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'])"

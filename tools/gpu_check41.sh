# eviction D2H overlap evidence (CUDA-event intervals on the side and main streams)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config c2 --p 0.2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_overlap.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2_overlap.log
grep '^{' gpurun_out/bench_c2_overlap.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['evict_compact']['evicted'], d['pcie'])"
tail -1 gpurun_out/bench_c2_overlap.log

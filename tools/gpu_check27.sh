cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 tools/pcie_probe/pcie_probe > gpurun_out/pcie_probe.json 2>&1
cat gpurun_out/pcie_probe.json
timeout 900 python bench.py --no-cpu-baseline --e2e-chunks 32 > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
python -c "
import json
for l in open('gpurun_out/bench_default.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'])
"

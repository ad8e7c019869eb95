# final lines for the remaining configs (C2 p=0.05, C3 max-length, C4 64k pool on one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config c2 --p 0.05 --no-cpu-baseline > gpurun_out/final_c2_p005.log 2>&1; echo "rc=$?" >> gpurun_out/final_c2_p005.log
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/final_c3.log 2>&1; echo "rc=$?" >> gpurun_out/final_c3.log
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/final_c4.log 2>&1; echo "rc=$?" >> gpurun_out/final_c4.log
for f in final_c2_p005 final_c3 final_c4; do grep '^{' gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', round(d['value']), round(d['ms_per_step'],2), round(r['frac'],3), d['config']['mean_batch'], d['evict_compact']['evicted'], round(d['e2e']['value']))"; tail -1 gpurun_out/$f.log; done

# DRAM traffic of the tensor-core attention launches on the exact LLaMA-3-8B bench command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_llama_final.csv python bench.py --shape llama3-8b --steps 30 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/ncu_llama_final.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_llama_final.log
tail -2 gpurun_out/ncu_llama_final.log
timeout 900 python bench.py --shape llama3-8b --steps 30 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_llama_k30.log 2>&1
grep '^{' gpurun_out/bench_llama_k30.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('alg bytes/launch', r['algorithmic_bytes_per_launch'], 'launches timed', d['steps'])"

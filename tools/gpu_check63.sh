# k_synth with per-row counter bases: generator parity (T0 checks inside lockstep) + timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c0_full_run or gptj_heads or grouped_query_kv or randomized" > gpurun_out/pytest_synth.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_synth.log
tail -2 gpurun_out/pytest_synth.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_synth -c 20 --csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep k_synth | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1
grep '^{' gpurun_out/bench_c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value']), d['ms_per_step'], d['phases_ms_per_step'])"

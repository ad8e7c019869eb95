# k_fill with counter bases: parity subset (arena rows byte-exact vs the oracle, P2 verify) + C1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c0_full_run or gptj_heads or grouped_query_kv or randomized or zero_length or bench_configuration_sampled" > gpurun_out/pytest_fill.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fill.log
tail -2 gpurun_out/pytest_fill.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1
grep '^{' gpurun_out/bench_c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value']), d['ms_per_step'], d['phases_ms_per_step'])"

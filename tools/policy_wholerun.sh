#!/usr/bin/env bash
# Whole-run allocation-policy comparison with the GPT-J random-weight proxy:
# every policy serves the same 8192-request pool to completion; tokens/s over the whole run.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in "--config c3 --steps 6000" "--config c1 --policy bucket --steps 1800" "--config c2 --p 0.05 --steps 1800" "--config c1 --steps 1800"; do
  name=$(echo $cfg | tr ' -' '__')
  timeout 1500 python bench.py --model gptj $cfg --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_whole$name.log 2>&1
  echo "$cfg rc=$?" >> gpurun_out/r02_whole$name.log
  grep '^{' gpurun_out/r02_whole$name.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$cfg', round(d['value']), 'tokens', d['tokens'], 'finished', d['finished'], 'mean_batch', round(d['config']['mean_batch'],1), 'ms/step', round(d['ms_per_step'],2), 'evicted', d['evict_compact']['evicted'])"
done

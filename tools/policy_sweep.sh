#!/usr/bin/env bash
# GPT-J proxy (random weights) around the S^3 path: ORCA-style max-length
# reservation vs bucket predictor vs S^3 with short mispredictions vs Oracle.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in "--config c3" "--config c1 --policy bucket" "--config c2 --p 0.05" "--config c1"; do
  name=$(echo $cfg | tr ' -' '__')
  timeout 900 python bench.py --model gptj $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02_sweep$name.log 2>&1
  echo "$cfg rc=$?" >> gpurun_out/r02_sweep$name.log
done

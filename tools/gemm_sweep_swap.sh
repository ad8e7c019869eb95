#!/usr/bin/env bash
# small-batch sweep of s3_gemm: swapped operands (W rows on the MMA's M side, the default
# for M <= 64) against the unswapped tiles (S3_GEMM_SWAP=0), with and without stream-K
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ms=${2:-1,8,16,32,48,64,96,128}
{
  for sw in 0 1; do
    S3_GEMM_SWAP=$sw timeout 300 python tools/gemm_bench.py --m $ms --iters 20 --copies 4 | sed "s/^{/{\"swap\": $sw, \"sk\": \"auto\", /"
  done
  S3_GEMM_SWAP=1 S3_GEMM_SK=0 timeout 300 python tools/gemm_bench.py --m $ms --iters 20 --copies 4 | sed "s/^{/{\"swap\": 1, \"sk\": 0, /"
} > gpurun_out/${1:-gemm_sweep_swap}.jsonl 2>&1

#!/usr/bin/env bash
# small-batch sweep of s3_gemm single-CTA tiles: tile width (S3_GEMM_BN) x stream-K (S3_GEMM_SK)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for bn in 64 128 256; do for sk in 0 1; do
  S3_GEMM_CG=1 S3_GEMM_BN=$bn S3_GEMM_SK=$sk timeout 300 python tools/gemm_bench.py --m 32,64,128,192,256 --iters 10 \
    | sed "s/^{/{\"bn\": $bn, \"sk\": $sk, /"
done; done > gpurun_out/${1:-gemm_sweep_small}.jsonl 2>&1

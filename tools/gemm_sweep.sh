#!/usr/bin/env bash
# tile-config sweep of s3_gemm: CTA group (S3_GEMM_CG) x stream-K (S3_GEMM_SK) at small / medium batches
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cg in 1 2; do for sk in 0 1; do
  S3_GEMM_CG=$cg S3_GEMM_SK=$sk timeout 300 python tools/gemm_bench.py --m 256,512,1024,2048 --iters 10 \
    | sed "s/^{/{\"cg\": $cg, \"sk\": $sk, /"
done; done > gpurun_out/${1:-gemm_sweep}.jsonl 2>&1

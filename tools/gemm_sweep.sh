#!/usr/bin/env bash
# tile-config sweep of s3_gemm: CTA group (S3_GEMM_CG) x split-K factor (S3_GEMM_S) at small batches
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cg in 1 2; do for sp in 1 2 3 4; do
  S3_GEMM_CG=$cg S3_GEMM_S=$sp timeout 300 python tools/gemm_bench.py --m 256,512,1024 --iters 10 \
    | sed "s/^{/{\"cg\": $cg, \"s\": $sp, /"
done; done > gpurun_out/${1:-gemm_sweep}.jsonl 2>&1

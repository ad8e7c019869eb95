#!/usr/bin/env bash
# stream-K reduction sweep of s3_gemm (CUDA-graph timing, weights cycled past L2):
# S3_GEMM_RED=1 (contributors TMA-reduce-add into one fp32 tile) vs 0 (one partial slot each,
# summed by the last group), stream-K as planned (auto) or forced on (S3_GEMM_SK=1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ms=${2:-8,64,128,161,256,512}
{
  for red in 0 1; do for sk in auto 1; do
    if [ $sk = auto ]; then unset S3_GEMM_SK; else export S3_GEMM_SK=$sk; fi
    S3_GEMM_RED=$red timeout 300 python tools/gemm_bench.py --m $ms --iters 20 --copies 4 --graph \
      | sed "s/^{/{\"red\": $red, \"sk\": \"$sk\", /"
  done; done
} > gpurun_out/${1:-gemm_sweep_red}.jsonl 2>&1

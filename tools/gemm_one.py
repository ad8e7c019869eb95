#!/usr/bin/env python
"""One s3_gemm shape, a few launches (a target for ncu):
    python tools/gemm_one.py --m 161 --shape o [--reps 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 2), "ffn_up": (16384, 4096, 1), "ffn_down": (4096, 16384, 2)}


def main():
    import torch
    from paper_2306_06000_b200 import s3 as abi
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=161)
    ap.add_argument("--shape", default="o", choices=sorted(SHAPES))
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    N, K, epi = SHAPES[args.shape]
    M = args.m
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    d = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(max(abi.s3_gemm_workspace(M, N, K, epi=epi), 16), device="cuda", dtype=torch.uint8)
    st = torch.cuda.current_stream()
    for _ in range(args.reps):
        abi.s3_gemm(st, a, w, d, c=d if epi == 2 else None, epi=epi, workspace=ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()

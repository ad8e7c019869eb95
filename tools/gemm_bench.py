#!/usr/bin/env python
"""TFLOP/s of libs3's tcgen05 GEMM (s3_gemm) on the GPT-J projection shapes
at batch M, beside cuBLAS (torch.matmul) on the same operands, against the
measured bf16 peak in MEASURED_PEAKS.json.  One JSON line per (M, shape).

    python tools/gemm_bench.py [--m 128,512,2048] [--iters 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 2), "ffn_up": (16384, 4096, 1), "ffn_down": (4096, 16384, 2)}


def main():
    import torch

    from paper_2306_06000_b200 import build
    from paper_2306_06000_b200 import s3 as abi
    build.build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", default="128,256,512,1024,2048,4096")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--copies", type=int, default=1,
                    help="cycle through this many weight copies (> L2 in total: weights streamed from HBM)")
    ap.add_argument("--graph", action="store_true",
                    help="time a CUDA graph of the iterations (device time without host launch gaps)")
    ap.add_argument("--lib", default=None, help="A/B: load this libs3.so build instead of the in-tree one")
    args = ap.parse_args()
    if args.lib:
        abi.LIB_PATH = os.path.abspath(args.lib)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for M in [int(x) for x in args.m.split(",")]:
        tot_flop, tot_ms, tot_ms_cb = 0.0, 0.0, 0.0
        for name, (N, K, epi) in SHAPES.items():
            a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            ws_ = [(torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16) for _ in range(args.copies)]
            w = ws_[0]
            it = [0]
            d = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            ws = torch.zeros(max(abi.s3_gemm_workspace(M, N, K, epi=epi), 16), device="cuda", dtype=torch.uint8)

            def nxt():
                it[0] += 1
                return ws_[it[0] % len(ws_)]

            def ours():
                abi.s3_gemm(st, a, nxt(), d, c=d if epi == 2 else None, epi=epi, workspace=ws)

            def cublas():
                torch.matmul(a, nxt().T, out=d)

            res = {}
            for tag, fn in (("s3_gemm", ours), ("cublas", cublas)):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                if args.graph:
                    gs = torch.cuda.Stream()
                    gs.wait_stream(torch.cuda.current_stream())
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.stream(gs):
                        stc = torch.cuda.current_stream()
                        with torch.cuda.graph(graph, stream=gs):
                            for _ in range(args.iters):
                                if tag == "s3_gemm":
                                    abi.s3_gemm(stc, a, nxt(), d, c=d if epi == 2 else None, epi=epi, workspace=ws)
                                else:
                                    fn()
                    torch.cuda.synchronize()
                    graph.replay()
                    torch.cuda.synchronize()
                    e0.record()
                    graph.replay()
                    e1.record()
                else:
                    e0.record()
                    for _ in range(args.iters):
                        fn()
                    e1.record()
                torch.cuda.synchronize()
                res[tag] = e0.elapsed_time(e1) / args.iters
            flop = 2.0 * M * N * K
            tf = flop / (res["s3_gemm"] / 1e3) / 1e12
            tf_cb = flop / (res["cublas"] / 1e3) / 1e12
            tot_flop += flop
            tot_ms += res["s3_gemm"]
            tot_ms_cb += res["cublas"]
            wbytes = 2.0 * N * K
            print(json.dumps({"M": M, "shape": name, "N": N, "K": K, "epi": epi, "us": round(res["s3_gemm"] * 1e3, 1),
                              "tflops": round(tf, 1), "frac_sustained": round(tf / peaks["bf16_tflops_sustained"], 3),
                              "weight_gbs": round(wbytes / (res["s3_gemm"] / 1e3) / 1e9, 1),
                              "cublas_us": round(res["cublas"] * 1e3, 1), "cublas_tflops": round(tf_cb, 1),
                              "vs_cublas": round(res["cublas"] / res["s3_gemm"], 3)}), flush=True)
        tf = tot_flop / (tot_ms / 1e3) / 1e12
        print(json.dumps({"M": M, "shape": "layer (qkv+o+ffn)", "tflops": round(tf, 1),
                          "frac_sustained": round(tf / peaks["bf16_tflops_sustained"], 3),
                          "cublas_tflops": round(tot_flop / (tot_ms_cb / 1e3) / 1e12, 1),
                          "vs_cublas": round(tot_ms_cb / tot_ms, 3)}), flush=True)


if __name__ == "__main__":
    main()

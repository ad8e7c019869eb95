#!/usr/bin/env python
"""Event-timed floor of one small kernel launch on a busy stream (the
harness overhead k_prep's CUDA-event time includes): CUDA events around
(a) nothing, (b) libs3's s3_cast_bf16 on 16 elements, with the stream kept
busy by matmuls so the launches are queued ahead of the GPU."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2306_06000_b200 import s3 as abi
    busy = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
    src = torch.zeros(16, device="cuda")
    dst = torch.zeros(16, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream()
    res = {"empty": [], "cast16": [], "cast16_x2": []}
    for it in range(12):
        for tag in res:
            for _ in range(10):
                busy @ busy
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if tag != "empty":
                abi.s3_cast_bf16(st, src, dst)
            if tag == "cast16_x2":
                abi.s3_cast_bf16(st, src, dst)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                res[tag].append(e0.elapsed_time(e1) * 1e3)
    for tag, v in res.items():
        v.sort()
        print(f"{tag}: median {v[len(v) // 2]:.2f} us, min {v[0]:.2f} us")


if __name__ == "__main__":
    main()

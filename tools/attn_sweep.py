"""Attention-kernel sweep over batch / length regimes (CUDA-event timing of
the decode step's attention launches through the C ABI).

Each case admits B requests with prompt length P (generous allocations so
nothing finishes or moves), then times `steps` decode steps.  Prints one
JSON line per case: attention GB/s (algorithmic bytes / kernel time) and
the fraction of the measured HBM copy peak."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_06000_b200.engine import S3Engine  # noqa: E402

CASES = [  # (name, L, H, Hkv, D, B, P, attn_variant)
    ("gptj long", 28, 16, 16, 256, 64, 1900),
    ("gptj mid", 28, 16, 16, 256, 1024, 200),
    ("gptj short", 28, 16, 16, 256, 4096, 24),
    ("gptj B=8", 28, 16, 16, 256, 8, 1900),
    ("llama3-8b gqa", 32, 32, 8, 128, 2048, 400),
    ("mqa H=16 D=128", 32, 16, 1, 128, 2048, 400),
    ("llama3-8b gqa tc", 32, 32, 8, 128, 2048, 400, 2),
    ("llama3-8b gqa tc short", 32, 32, 8, 128, 8192, 40, 2),
    ("mqa H=16 D=128 tc", 32, 16, 1, 128, 2048, 400, 2),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--case", default=None, help="run only cases whose name contains this")
    ap.add_argument("--lib", default=None, help="A/B: load this libs3.so build instead of the in-tree one")
    ap.add_argument("--chunk", type=int, default=0, help="split-K unit rows C (0: the library default, 512)")
    ap.add_argument("--custom", action="append", default=[],
                    help="extra case 'name:L,H,Hkv,D,B,P,variant' (repeatable)")
    args = ap.parse_args()
    for c in args.custom:
        name, vals = c.split(":")
        v = [int(x) for x in vals.split(",")]
        CASES.append((name, *v))
    if args.lib:
        from paper_2306_06000_b200 import s3 as abi
        abi.LIB_PATH = os.path.abspath(args.lib)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for case in CASES:
        name, L, H, Hkv, D, B, P = case[:7]
        if args.case and args.case not in name:
            continue
        variant = case[7] if len(case) > 7 else 0
        kvpt = 4 * L * Hkv * D
        R = max(2048, B * (P + args.steps + 8))
        if R * kvpt > 150e9:
            continue
        eng = S3Engine(L, H, D, 2048, R, max(B, 16), num_kv_heads=0 if Hkv == H else Hkv,
                       host_store_bytes=64 << 20, attn_variant=variant, chunk_rows=args.chunk)
        n = B
        eng.submit(np.arange(n), np.full(n, P), np.full(n, args.steps + 8), np.full(n, 10_000))
        eng.admit()
        eng.step()
        eng.profile(True)
        for _ in range(args.steps):
            eng.step()
        p = eng.profile_get()
        gbs = (p.attn_bytes + p.fused_move_bytes) / (p.attn_ms / 1e3) / 1e9
        print(json.dumps({"case": name, "chunk": args.chunk or 512, "L": L, "H": H, "Hkv": Hkv, "D": D, "B": B, "len": P,
                          "attn_ms_per_step": round(p.attn_ms / args.steps, 4), "gbs": round(gbs, 1),
                          "frac_of_peak": round(gbs / peak, 3)}), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

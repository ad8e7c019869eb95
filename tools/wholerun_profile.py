#!/usr/bin/env python
"""Attention throughput along a whole run (diagnostic): the C1 workload of a
bench shape from the first admission until every request finished, with the
attention kernel's CUDA-event time and algorithmic bytes read every `--every`
steps (s3_profile deltas), beside the batch size and mean resident rows.

    python tools/wholerun_profile.py [--shape llama3-8b] [--requests 32768] [--every 50]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import s3synth
    from bench import GPTJ, SHAPES
    from paper_2306_06000_b200.engine import S3Engine
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama3-8b", choices=sorted(SHAPES))
    ap.add_argument("--requests", type=int, default=32768)
    ap.add_argument("--every", type=int, default=50)
    args = ap.parse_args()
    shp = SHAPES[args.shape]
    L, H, D, Hkv = shp["L"], shp["H"], shp["D"], shp["Hkv"]
    kvpt = 4 * L * Hkv * D
    t = s3synth.make_trace(args.requests, seed=1, policy="oracle", max_seq_len=GPTJ["max_len"])
    max_running = 16384 if Hkv < H else 8192
    free_b, _ = torch.cuda.mem_get_info()
    io = max_running * L * D * (H * 2 + 2 * Hkv * 2 + H * 4)
    R = int((free_b - io - (4 << 30) - (8 << 30)) // kvpt)
    variant = 2 if (Hkv < H and D == 128) else 0
    eng = S3Engine(L, H, D, GPTJ["max_len"], R, max_running, num_kv_heads=0 if Hkv == H else Hkv,
                   staging_bytes=4 << 30, host_store_bytes=1 << 30, attn_variant=variant)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    eng.profile(True)
    prev = eng.profile_get()
    step, rows_acc, b_acc, n_acc = 0, 0, 0, 0
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.9
    while True:
        c = eng.counters_local()
        if eng.B == 0 and c[3] + c[4] == 0:
            break
        bv = eng.batch_view()
        b_acc += len(bv)
        rows_acc += sum(s[3] + 1 for s in bv)
        n_acc += 1
        eng.step()
        step += 1
        if step % args.every == 0:
            p = eng.profile_get()
            ms = p.attn_ms - prev.attn_ms
            by = (p.attn_bytes + p.fused_move_bytes) - (prev.attn_bytes + prev.fused_move_bytes)
            print(json.dumps({"steps": f"{step - args.every}..{step - 1}", "mean_B": round(b_acc / n_acc, 1),
                              "mean_rows": round(rows_acc / max(b_acc, 1), 1),
                              "attn_ms_per_step": round(ms / args.every, 3),
                              "frac": round(by / (ms / 1e3) / 1e9 / peak, 3) if ms else None}), flush=True)
            prev, b_acc, n_acc, rows_acc = p, 0, 0, 0
    eng.close()


if __name__ == "__main__":
    main()

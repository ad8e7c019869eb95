#!/usr/bin/env python
"""k_prep (detection + keep-scan + work list) at large batches: B tiny
sequences (L = 1, H = 1, D = 64, so the attention pass is negligible), run
under `ncu --metrics gpu__time_duration.sum -k regex:k_prep` to time the
scan kernel alone (single CTA up to 2048 slots, one CTA per 512 above).

    python tools/prep_bench.py [B] [p]      p: share of under-predicted requests (0.2)
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import s3synth
    from paper_2306_06000_b200 import s3 as abi
    from paper_2306_06000_b200.engine import S3Engine
    if os.environ.get("S3_LIB"):                     # A/B: another libs3.so build (e.g. -DPREP_TRACE)
        abi.LIB_PATH = os.path.abspath(os.environ["S3_LIB"])
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2      # share of under-predicted requests
    t = s3synth.make_trace(B, seed=3, policy="short", p=p, max_seq_len=64, prompt_max=16)
    eng = S3Engine(1, 1, 64, 64, int(t.cap.sum()) + 64, B, host_store_bytes=1 << 26)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    busy = torch.randn(4096, 4096, device="cuda").to(torch.bfloat16)
    eng.profile(True)
    for _ in range(8):
        for _ in range(20):                          # keep the SM clocks up between steps
            busy @ busy
        eng.synth_inputs()
        ev0.record()
        eng.decode()
        ev1.record()
        torch.cuda.synchronize()
        print(f"B {eng.B}: decode call (k_prep + k_deps + attention) {ev0.elapsed_time(ev1) * 1e3:.1f} us")
        eng.evict_compact()
        eng.admit()
    pr = eng.profile_get()
    print(f"k_prep (CUDA events around each launch): {pr.prep_ms * 1e3 / max(pr.prep_launches, 1):.1f} us "
          f"mean over {pr.prep_launches} launches")
    eng.close()


if __name__ == "__main__":
    main()

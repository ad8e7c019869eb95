"""Per-role timeline of the tensor-core kernel's tiles on CTA 0 (diagnostic;
needs a -DTC_TRACE build of libs3.so: the build.py nvcc line with -DTC_TRACE).

Slots (SM clock): 0 producer got a stage, 1 producer issued the tile's loads,
2 softmax finished the item's epilogue (last tiles), 3 MMA saw the tile land, 4 MMA got P, 5 MMA committed O, 6 softmax got S,
7 softmax handed over P."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", required=True)
    ap.add_argument("--B", type=int, default=8192)
    ap.add_argument("--P", type=int, default=40)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--groups", type=int, default=2, help="softmax groups of the traced build (NG)")
    args = ap.parse_args()
    from paper_2306_06000_b200 import s3 as abi
    abi.LIB_PATH = os.path.abspath(args.lib)
    from paper_2306_06000_b200.engine import S3Engine
    L, H, Hkv, D = 32, 32, 8, 128
    R = max(2048, args.B * (args.P + args.steps + 8))
    eng = S3Engine(L, H, D, 2048, R, args.B, num_kv_heads=Hkv, host_store_bytes=64 << 20, attn_variant=2)
    n = args.B
    eng.submit(np.arange(n), np.full(n, args.P), np.full(n, args.steps + 8), np.full(n, 10_000))
    eng.admit()
    for _ in range(args.steps):
        eng.step()
    import torch
    torch.cuda.synchronize()
    N = 8192 * 8
    buf = (C.c_ulonglong * N)()
    rc = abi.lib().s3_debug_tc_trace(buf, N)
    assert rc == 0, rc
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.int64)
    valid = (tr[:, 5] > 0) & (tr[:, 0] > 0) & (tr[:, 6] > 0)
    idx = np.nonzero(valid)[0]
    idx = idx[(idx > 16) & (idx < idx.max() - 16)]
    idx = idx[tr[idx + args.groups, 6] > 0]
    t = tr[idx]
    per = np.diff(tr[idx, 5])
    res = {
        "tiles": int(len(idx)),
        "period_cycles_median": float(np.median(per)),
        "producer_wait_stage_to_issue_end": float(np.median(t[:, 1] - t[:, 0])),
        "issue_end_to_landed(MMA saw)": float(np.median(t[:, 3] - t[:, 1])),
        "landed_to_softmax_got_S": float(np.median(t[:, 6] - t[:, 3])),
        "softmax_S_to_P": float(np.median(t[:, 7] - t[:, 6])),
        "P_handover_to_MMA_got_P": float(np.median(t[:, 4] - t[:, 7])),
        "MMA_got_P_to_O_committed": float(np.median(t[:, 5] - t[:, 4])),
        "stage_reuse_gap(O commit t -> producer got stage t+3)": float(np.median(tr[idx + 3, 0] - t[:, 5])),
        "issue_end_t_to_stage_t+1": float(np.median(tr[idx + 1, 0] - t[:, 1])),
    }
    # per-tile stage life and occupancy from the raw timestamps (CTA 0)
    life = t[:, 5] - t[:, 0]
    span = float(t[:, 5].max() - t[:, 0].min())
    res["stage_life_mean"] = float(life.mean())
    res["period_mean"] = span / len(idx)
    res["tiles_in_flight_mean"] = float(life.sum()) / span
    # gaps where the producer held no stage: got-stage(t+1) minus issue-end(t), split by whether t+1
    # starts a new (unit, layer) ticket (slot-0 of t+1 after an atomic) -- flags not traced, so report all
    res["producer_gap_p90"] = float(np.percentile(tr[idx + 1, 0] - t[:, 1], 90))
    res["softmax_group_busy_frac"] = float(((t[:, 7] - t[:, 6]).sum()) / span / 2)
    # short items (one tile per item): tile t belongs to softmax group t % groups; slot 2 = its
    # epilogue end.  Per group: S -> P, P -> epilogue end, and the idle gap until the group's
    # next S (waiting for the MMA thread / the ring)
    ep = tr[idx, 2]
    if (ep > 0).mean() > 0.9:
        res["group_S_to_P"] = float(np.median(t[:, 7] - t[:, 6]))
        res["group_P_to_epilogue_end"] = float(np.median(ep - t[:, 7]))
        nxt = tr[idx + args.groups, 6]
        res["group_idle_epilogue_end_to_next_S"] = float(np.median(nxt - ep))
        res["group_busy_frac"] = float(((ep - t[:, 6]).sum()) / span / args.groups)
        res["MMA_got_P_to_epilogue_end"] = float(np.median(ep - t[:, 4]))
        res["O_commit_to_epilogue_end"] = float(np.median(ep - t[:, 5]))
    print(json.dumps(res))
    eng.close()


if __name__ == "__main__":
    main()

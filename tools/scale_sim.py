#!/usr/bin/env python
"""Length-only replay of the sequence-partitioned multi-GPU decode loop.

Why: with one process per GPU in lockstep, a step lasts as long as the
busiest rank's attention pass, which streams sum_b (len_b + 1) KV rows
(DESIGN.md §9).  This replay tracks only lengths -- no KV values -- and
reports the bytes-weighted lockstep efficiency

    eff = sum_t mean_r rows_r(t) / sum_t max_r rows_r(t),   rows_r = sum_b (len_b + 1)

for the multi-bin FFD placement rules of DESIGN.md R26:
  * "first": each item to the first rank (in rank order) with room  (round 1);
  * "worst": each item to the rank with the most free rows, ties to the
             lowest rank (worst fit; the current rule).

The step mirrors the library's order: decode (len += 1) -> detect (EOS,
length stop at max_len R28, overrun at len == cap) -> evict (home queue,
cap doubled, R5) + compact (tail = sum of kept caps) -> per rank, re-admit
own evicted requests (local FFD) -> multi-bin FFD of the shared fresh pool
(free rows = R - tail, free slots = max_running - B).

    python tools/scale_sim.py                 # the driver's weak-scaling runs
    python tools/scale_sim.py --quick         # smaller pools (what the test runs)
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import s3synth  # noqa: E402

GPTJ_R = 367446          # arena rows per GPU in the bench (168.6 GB of GPT-J KV)
MAX_RUNNING = 8192


class CapPool:
    """Requests waiting for admission, in FFD order (cap desc, req asc), with
    the query "largest cap <= f, smallest req among those" in O(max_len)."""

    def __init__(self, max_len):
        self.q = [[] for _ in range(max_len + 1)]     # per cap: req ids ascending (appended in order)
        self.head = np.zeros(max_len + 1, np.int64)
        self.count = np.zeros(max_len + 1, np.int64)
        self.n = 0

    def add(self, caps, reqs):
        order = np.lexsort((reqs, -caps))
        for c, r in zip(caps[order], reqs[order]):
            self.q[c].append(int(r))
            self.count[c] += 1
        self.n += len(caps)

    def add_one(self, cap, req):
        lst = self.q[cap]
        lst.insert(int(np.searchsorted(np.asarray(lst[self.head[cap]:], np.int64), req)) + int(self.head[cap]), req)
        self.count[cap] += 1
        self.n += 1

    def largest_le(self, f):
        f = min(int(f), len(self.count) - 1)
        if f <= 0:
            return -1
        nz = np.flatnonzero(self.count[1:f + 1])
        return int(nz[-1]) + 1 if nz.size else -1

    def items(self):
        """(caps, reqs) of every waiting item."""
        caps, reqs = [], []
        for c in np.flatnonzero(self.count):
            q = self.q[c][self.head[c]:]
            caps += [int(c)] * len(q)
            reqs += q
        return np.array(caps, np.int64), np.array(reqs, np.int64)

    def pop(self, cap):
        r = self.q[cap][self.head[cap]]
        self.head[cap] += 1
        self.count[cap] -= 1
        self.n -= 1
        return r


class Rank:
    def __init__(self, R, max_running):
        self.R, self.max_running = R, max_running
        self.req = np.zeros(0, np.int64)
        self.len = np.zeros(0, np.int64)
        self.cap = np.zeros(0, np.int64)
        self.gen = np.zeros(0, np.int64)
        self.tail = 0
        self.home = None

    @property
    def B(self):
        return self.req.shape[0]

    def place(self, reqs, lens, caps, gens):
        self.req = np.concatenate([self.req, np.asarray(reqs, np.int64)])
        self.len = np.concatenate([self.len, np.asarray(lens, np.int64)])
        self.cap = np.concatenate([self.cap, np.asarray(caps, np.int64)])
        self.gen = np.concatenate([self.gen, np.asarray(gens, np.int64)])
        self.tail += int(np.sum(caps))


def choose(rule, free, slots, cap):
    ok = slots > 0
    if not ok.any():
        return -1
    if rule == "first":
        cand = np.flatnonzero(ok & (free >= cap))
        return int(cand[0]) if cand.size else -1
    f = np.where(ok, free, -1)
    r = int(np.argmax(f))                         # ties: lowest rank
    return r if f[r] >= cap else -1


def multibin_ffd(pool, free, slots, rule):
    """Assign pool items (FFD order) to ranks; returns [(rank, cap, req)]."""
    out = []
    free = free.copy()
    slots = slots.copy()
    while pool.n:
        ok = slots > 0
        if not ok.any():
            break
        mf = int(free[ok].max())
        c = pool.largest_le(mf)
        if c < 0:
            break
        # an item skipped here fits no rank now and never will this step (free only shrinks)
        r = choose(rule, free, slots, c)
        if r < 0:
            break
        req = pool.pop(c)
        free[r] -= c
        slots[r] -= 1
        out.append((r, c, req))
    return out


def simulate(n_req, G, rule, policy="oracle", p=0.0, R=GPTJ_R, max_running=MAX_RUNNING, seed=1,
             max_len=2048, window=(5, 25), max_steps=100000, check_plan=None):
    t = s3synth.make_trace(n_req, seed=seed, policy=policy, p=p, max_seq_len=max_len)
    P = t.prompt.astype(np.int64)
    O = t.out.astype(np.int64)
    pool = CapPool(max_len)
    pool.add(t.cap.astype(np.int64), t.req_id.astype(np.int64))
    ranks = [Rank(R, max_running) for _ in range(G)]
    homes = [CapPool(max_len) for _ in range(G)]
    host = [dict() for _ in range(G)]                # evicted req -> (len, gen)

    def admit_all(step):
        for r, rk in enumerate(ranks):               # local FFD of own evicted requests
            h = homes[r]
            while h.n and rk.B < max_running:
                c = h.largest_le(R - rk.tail)
                if c < 0:
                    break
                q = h.pop(c)
                ln, gn = host[r].pop(q)
                rk.place([q], [ln], [c], [gn])
        free = np.array([R - rk.tail for rk in ranks], np.int64)
        slots = np.array([max_running - rk.B for rk in ranks], np.int64)
        snap = pool.items() if check_plan is not None and check_plan(step, None, None, None, None) else None
        plan = multibin_ffd(pool, free, slots, rule)
        if snap is not None:
            check_plan(step, free, slots, snap, plan)
        per = [[] for _ in range(G)]
        for r, c, q in plan:
            per[r].append((q, c))
        for r, items in enumerate(per):
            if items:
                qs = np.array([q for q, _ in items], np.int64)
                ranks[r].place(qs, P[qs], [c for _, c in items], np.zeros(len(items), np.int64))

    admit_all(-1)
    rows_hist = []
    step = 0
    while step < max_steps:
        if pool.n == 0 and all(rk.B == 0 and homes[i].n == 0 for i, rk in enumerate(ranks)):
            break
        rows = np.array([int(np.sum(rk.len + 1)) if rk.B else 0 for rk in ranks], np.int64)
        rows_hist.append(rows)
        for r, rk in enumerate(ranks):
            if not rk.B:
                continue
            rk.len += 1
            rk.gen += 1
            fin = (rk.gen == O[rk.req]) | (rk.len >= max_len)
            ovr = ~fin & (rk.len == rk.cap)
            for i in np.flatnonzero(ovr):
                q = int(rk.req[i])
                host[r][q] = (int(rk.len[i]), int(rk.gen[i]))
                homes[r].add_one(int(min(2 * rk.cap[i], max_len)), q)
            keep = ~(fin | ovr)
            rk.req, rk.len, rk.cap, rk.gen = rk.req[keep], rk.len[keep], rk.cap[keep], rk.gen[keep]
            rk.tail = int(np.sum(rk.cap))
        admit_all(step)
        step += 1
    H = np.array(rows_hist, np.float64)
    mx = H.max(axis=1)
    mean = H.mean(axis=1)
    w0, w1 = window
    win = slice(w0, min(w1, H.shape[0]))
    return dict(G=G, rule=rule, policy=policy, steps=step,
                eff_run=float(mean.sum() / mx.sum()),
                eff_window=float(mean[win].sum() / mx[win].sum()) if mx[win].sum() else 1.0,
                median_max_over_mean=float(np.median(mx[mean > 0] / mean[mean > 0])))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="1/4-size pools and arenas")
    ap.add_argument("--per-gpu", type=int, default=8192)
    ap.add_argument("--gpus", default="2,4,8")
    ap.add_argument("--policies", default="oracle,bucket")
    a = ap.parse_args()
    scale = 4 if a.quick else 1
    for policy in a.policies.split(","):
        for G in [int(x) for x in a.gpus.split(",")]:
            res = {rule: simulate(a.per_gpu // scale * G, G, rule, policy=policy, R=GPTJ_R // scale,
                                  max_running=MAX_RUNNING // scale) for rule in ("first", "worst")}
            f, w = res["first"], res["worst"]
            print(f"{policy:7s} G={G}: lockstep efficiency whole run  first-fit {f['eff_run']:.3f}  "
                  f"worst-fit {w['eff_run']:.3f} | driver window (steps 5-24) {f['eff_window']:.3f} -> "
                  f"{w['eff_window']:.3f} | steps {f['steps']} / {w['steps']}", flush=True)


if __name__ == "__main__":
    main()

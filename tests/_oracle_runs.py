"""Helpers that drive the oracle state machine over a trace (test infra)."""
from __future__ import annotations

import numpy as np

import oracle


def run_oracle(trace, L=1, H=1, D=8, R=None, max_running=1 << 20, seed=1, record=None,
               max_steps=100000):
    """Run a trace to completion on one oracle; returns a summary dict.

    record(step, o, rep, perm, ev, fin, admitted, pre_batch) is called each step.
    """
    R = R if R is not None else trace.max_seq_len
    o = oracle.Oracle(L, H, D, trace.max_seq_len, R, max_running=max_running, seed=seed)
    o.submit(trace.req_id, trace.prompt, trace.alloc)
    admitted0 = o.admit()
    out = dict(steps=0, batch_sizes=[], d2h=0, moved=0, evictions={}, evict_gens={},
               admitted0=admitted0, paper_pcie=0, paper_hbm=0, finished_step={})
    step = 0
    while True:
        c = o.counters()
        if o.B == 0 and c[3] + c[4] == 0:
            break
        if step >= max_steps:
            raise RuntimeError("run did not terminate")
        pre = o.batch()
        out["batch_sizes"].append(len(pre))
        q, k, v, eos = o.make_inputs(trace.out)
        o.decode(q, k, v, eos)
        rep, perm, ev, fin = o.evict_compact()
        out["d2h"] += rep.d2h_bytes
        out["moved"] += rep.moved_bytes
        out["paper_pcie"] += rep.paper_pcie_bytes
        out["paper_hbm"] += rep.paper_hbm_bytes
        for e in ev:
            out["evictions"][e[0]] = out["evictions"].get(e[0], 0) + 1
            out["evict_gens"].setdefault(e[0], []).append(e[3])
        for r in fin:
            out["finished_step"][int(r)] = step
        adm = o.admit()
        if record is not None:
            record(step, o, rep, perm, ev, fin, adm, pre)
        step += 1
    out["steps"] = step
    out["oracle"] = o
    return out


def expected_evictions(cap0: int, P: int, O: int, max_len: int):
    """P3 closed form: request r is evicted k_r = min{k >= 0 : min(cap0 2^k, max_len)
    >= P+O} times, the j-th time at gen = min(cap0 2^j, max_len) - P."""
    gens = []
    c = cap0
    while c < P + O:
        gens.append(c - P)
        c = min(2 * c, max_len)
    return gens

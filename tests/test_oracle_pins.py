"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Every test names the pin (DESIGN.md "Oracle pins" P1..P9) and the passage.
"""
from __future__ import annotations

import itertools
import math
import os

import numpy as np
import pytest
import torch

import oracle
import s3synth
from tests._oracle_runs import expected_evictions, run_oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------------------
# Paper-printed values and closed forms
# ---------------------------------------------------------------------------

def test_kv_bytes_per_token_paper_values(oracle_lib):
    # PAPER.md:111 [§2.1]: GPT-NEOX, 44 layers, 6144 hidden -> "1MB per KV cache per token"
    neox = oracle.kv_bytes_per_token(44, 64, 96)
    assert neox == 1_081_344
    assert abs(neox - 2**20) / 2**20 < 0.04
    # PAPER.md:127 [§2.2]: 2048 tokens -> "2.2GB per sequence"
    assert neox * 2048 == 2_214_592_512
    assert round(neox * 2048 / 1e9, 1) == 2.2
    # 80 GB A100, 40 GB model -> "less than 20" max-length sequences
    assert (80e9 - 40e9) // (neox * 2048) < 20
    # GPT-J (d = 16 x 256 = 4096, R3)
    assert oracle.kv_bytes_per_token(28, 16, 256) == 458_752
    # SPEC.md:63 unit case: l = 1, d_h = 1 -> 4 bytes
    assert oracle.kv_bytes_per_token(1, 1, 1) == 4


def test_eviction_penalty_worked_example(oracle_lib):
    # SPEC.md:289 worked example of PAPER.md:15: resident 8 B, BW_H2D 2 B/s,
    # rows below 4 B, BW_HBM 4 B/s -> 2(8/2 + 4/4) = 10 s
    assert oracle.eviction_penalty(8, 4, 2, 4) == pytest.approx(10.0)
    # evicting the last row -> no rearrangement term
    assert oracle.eviction_penalty(8, 0, 2, 4) == pytest.approx(8.0)


def test_pool_penalty_insights(oracle_lib):
    # "the eviction penalty does not exist as long as the
    # predictor does not make any short predictions": p = 0 -> 0
    assert oracle.pool_penalty(0.0, 1e6, 1e9, 1e11, 1e9, 1e12) == 0.0
    # SPEC.md:300 worked example: p=.5, N=2, mean S_P 8, sum 4, BW 2 / 4 -> 9 s
    assert oracle.pool_penalty(0.5, 2, 8, 4, 2, 4) == pytest.approx(9.0)
    # PAPER.md:26 "dependent only on the memory bandwidths": doubling both halves it
    a = oracle.pool_penalty(0.1, 1000, 3e7, 5e9, 25e9, 6.4e12)
    b = oracle.pool_penalty(0.1, 1000, 3e7, 5e9, 50e9, 12.8e12)
    assert b == pytest.approx(a / 2)


def test_pool_penalty_is_mean_of_event_penalties(oracle_lib):
    # with the evicted row uniform over the n resident rows,
    # the expected rows-below sum is half the resident total ("We read on
    # average m/2 rows"), so the pool formula equals p N times the average of
    # the per-event formula over positions, up to the (n-1)/n discrete term.
    rng = np.random.default_rng(3)
    n = 4000
    sp = rng.integers(50, 250, n).astype(float)
    bw_h, bw_m = 25e9, 6.4e12
    below = np.concatenate([np.cumsum(sp[::-1])[::-1][1:], [0.0]])
    per_event = np.mean([oracle.eviction_penalty(sp[i], below[i], bw_h, bw_m) for i in range(n)])
    pool = oracle.pool_penalty(1.0, 1, sp.mean(), sp.sum(), bw_h, bw_m)
    assert per_event == pytest.approx(pool, rel=2e-3)


def test_underutilization_ratio(oracle_lib):
    # ratio = sum S_A / sum S_P; the oracle predictor -> 1.
    t = s3synth.make_trace(20000, seed=1, policy="oracle")
    sa = (t.prompt + t.out).astype(np.int64)
    assert oracle.underutilization_ratio(sa, t.cap) == 1.0
    # max-length allocation "suffers from massive underutilization"
    tm = s3synth.make_trace(20000, seed=1, policy="maxlen")
    r_max = oracle.underutilization_ratio(sa, tm.cap)
    assert np.all(tm.cap == 2048)
    assert r_max == pytest.approx(sa.sum() / (2048 * 20000))
    assert 0.04 < r_max < 0.08          # SURVEY.md §8(d) calibration: 0.0586
    tb = s3synth.make_trace(20000, seed=1, policy="bucket")
    r_b = oracle.underutilization_ratio(sa, tb.cap)
    assert r_max < r_b < 1.0
    # SPEC.md:446 scale invariance: multiplying all sizes by kvpt changes nothing
    kv = 458_752
    assert oracle.underutilization_ratio(sa * kv, tb.cap * kv) == pytest.approx(r_b, rel=1e-12)


# ---------------------------------------------------------------------------
# Generator (T0): C oracle == numpy reference == splitmix64 test vector
# ---------------------------------------------------------------------------

def test_splitmix64_test_vector(oracle_lib):
    # First output of SplitMix64 seeded with 0 (the published reference value).
    assert oracle.lib().s3o_splitmix64(0) == 0xE220A8397B1DCDAF
    assert int(s3synth.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    xs = np.array([1, 2, 12345, 2**63 + 7, 2**64 - 1], np.uint64)
    ref = s3synth.splitmix64(xs)
    for x, r in zip(xs, ref):
        assert oracle.lib().s3o_splitmix64(int(x)) == int(r)


@pytest.mark.parametrize("shape", [(1, 2, 64, 64), (28, 16, 256, 2048)])
def test_generator_matches_numpy(oracle_lib, shape):
    L, H, D, M = shape
    for (req, l, kv, pos) in [(0, 0, 0, 0), (7, L - 1, 1, M - 1), (65535, L // 2, 1, 5)]:
        c = oracle.gen_kv(L, H, D, M, 1, req, l, kv, pos)
        ref = s3synth.kv_elements(1, req, l, kv, pos, L, H, D, M)
        assert np.array_equal(oracle.bf16_bits_to_f64(c), ref)
        cq = oracle.gen_q(L, H, D, M, 1, req, l, pos)
        refq = s3synth.q_elements(1, req, l, pos, L, H, D, M)
        assert np.array_equal(oracle.bf16_bits_to_f64(cq), refq)
    # value range and exactness: k8/128 in [-1, 127/128]
    assert ref.min() >= -1.0 and ref.max() <= 127 / 128


# ---------------------------------------------------------------------------
# P1 attention special cases, and a library cross-check
# ---------------------------------------------------------------------------

def _one_step(L, H, D, max_len, R, prompts, allocs, seed=1, q=None, k=None, v=None):
    o = oracle.Oracle(L, H, D, max_len, R, seed=seed)
    n = len(prompts)
    o.submit(np.arange(n), prompts, allocs)
    o.admit()
    outs = np.full(n, 10_000, np.int32)
    q0, k0, v0, eos = o.make_inputs(outs)
    q = q0 if q is None else q
    k = k0 if k is None else k
    v = v0 if v is None else v
    out, st = o.decode(q, k, v, eos)
    return o, out, (q, k, v)


def test_attention_p0_first_token_is_v_new(oracle_lib):
    # P1(i): a request with P = 0 attends only to its own new row:
    # softmax = [1] so o = v_new exactly (R1).
    o, out, (q, k, v) = _one_step(2, 4, 64, 64, 64, [0, 0, 3], [5, 9, 4])
    p0 = [b for b, s in enumerate(o.batch()) if s[1] == 0]
    assert len(p0) == 2
    for b in p0:
        assert np.array_equal(out[:, b], oracle.bf16_bits_to_f64(v[:, b]))


def test_attention_zero_query_is_mean_of_values(oracle_lib):
    # P1(ii): q = 0 -> all scores equal -> o = mean of V rows 0..pos.
    o, _, (q, k, v) = _one_step(1, 2, 64, 64, 64, [5, 9], [3, 3])
    o2 = oracle.Oracle(1, 2, 64, 64, 64)
    o2.submit(np.arange(2), [5, 9], [3, 3])
    o2.admit()
    qz = np.zeros_like(q)
    out, _ = o2.decode(qz, k, v, np.zeros(2, np.uint8))
    A = o2.arena()
    for b, (req, P, gen, ln, cap, off) in enumerate(o2.batch()):
        rows = oracle.bf16_bits_to_f64(A[off:off + ln, 0, 1])    # [len, H, D] incl. new row
        assert np.allclose(out[0, b], rows.mean(axis=0), rtol=0, atol=1e-15)


def test_attention_equal_keys_uniform_weights(oracle_lib):
    # P1(iii): all K rows equal -> uniform softmax regardless of q.
    o = oracle.Oracle(1, 1, 64, 64, 64)
    o.submit(np.arange(1), [6], [3])
    o.admit()
    A = o.arena()
    A[0:6, 0, 0] = A[0, 0, 0]          # make the prompt keys identical
    q, k, v, eos = o.make_inputs(np.array([100], np.int32))
    k[0, 0] = A[0, 0, 0]
    out, _ = o.decode(q, k, v, eos)
    rows = oracle.bf16_bits_to_f64(o.arena()[0:7, 0, 1])
    assert np.allclose(out[0, 0], rows.mean(axis=0), rtol=0, atol=1e-15)


def test_attention_matches_torch_sdpa_fp64(oracle_lib):
    # P1(iv): library cross-check -- torch SDPA in fp64 on the same rows.
    L, H, D = 2, 4, 64
    prompts, allocs = [1, 7, 20, 33], [4, 4, 4, 4]
    o = oracle.Oracle(L, H, D, 64, 128)
    o.submit(np.arange(4), prompts, allocs)
    o.admit()
    q, k, v, eos = o.make_inputs(np.full(4, 100, np.int32))
    out, _ = o.decode(q, k, v, eos)
    A = o.arena()
    for b, (req, P, gen, ln, cap, off) in enumerate(o.batch()):
        for l in range(L):
            K = torch.from_numpy(oracle.bf16_bits_to_f64(A[off:off + ln, l, 0])).permute(1, 0, 2)
            V = torch.from_numpy(oracle.bf16_bits_to_f64(A[off:off + ln, l, 1])).permute(1, 0, 2)
            Q = torch.from_numpy(oracle.bf16_bits_to_f64(q[l, b]))[:, None, :]
            ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V)[:, 0, :].numpy()
            assert np.allclose(out[l, b], ref, rtol=0, atol=1e-12)


def test_attention_sharp_query_selects_row(oracle_lib):
    # P1(v): scaling one key far above the others makes softmax one-hot.
    o = oracle.Oracle(1, 1, 64, 64, 64)
    o.submit(np.arange(1), [10], [3])
    o.admit()
    A = o.arena()
    q, k, v, eos = o.make_inputs(np.array([100], np.int32))
    qv = np.zeros(64, np.float32); qv[0] = 256.0
    q[0, 0, 0] = (qv.view(np.uint32) >> 16).astype(np.uint16)
    kv = np.zeros((11, 64), np.float32); kv[:, 0] = -1.0; kv[4, 0] = 127 / 128   # row 4 wins by ~63
    bits = (kv.view(np.uint32) >> 16).astype(np.uint16)
    A[0:10, 0, 0, 0] = bits[:10]
    k[0, 0, 0] = bits[10]
    out, _ = o.decode(q, k, v, eos)
    s = 256.0 * kv[:, 0].astype(np.float64) / 8.0
    w = np.exp(s - s.max()); w /= w.sum()
    assert w[4] > 0.99
    V = oracle.bf16_bits_to_f64(o.arena()[0:11, 0, 1, 0])
    assert np.allclose(out[0, 0, 0], w @ V, atol=1e-14)


# ---------------------------------------------------------------------------
# C0 golden trace -- an independent hand computation
# ---------------------------------------------------------------------------

def _parse_golden():
    rows = []
    with open(os.path.join(GOLDEN, "c0_events.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


def test_c0_golden_events(oracle_lib):
    t = s3synth.c0_trace()
    events = {"admit": {}, "finish": {}, "evict": {}, "move": {}}
    pre_offs = {}

    def rec(step, o, rep, perm, ev, fin, adm, pre):
        offs = {s[0]: s[5] for s in o.batch()}
        if adm:
            events["admit"][step] = [f"{r}@{offs[r]}" for r in adm]
        if len(fin):
            events["finish"][step] = sorted(int(x) for x in fin)
        if ev:
            events["evict"][step] = (ev, rep, list(perm))
        moves = []
        for s in pre:
            r = s[0]
            if r in offs and offs[r] != s[5] and r not in [a for a in adm]:
                moves.append(f"{r}:{s[5]}->{offs[r]}:{s[3] + 1}")
        if moves:
            events["move"][step] = moves

    res = run_oracle(t, L=1, H=2, D=64, R=64, record=rec)
    o = res["oracle"]
    for kind, step, *fields in _parse_golden():
        if kind == "admit" and step == "init":
            assert [int(x.split("@")[0]) for x in fields] == res["admitted0"]
        elif kind == "admit":
            assert events["admit"][int(step)] == fields
        elif kind == "finish":
            assert events["finish"][int(step)] == [int(x) for x in fields]
        elif kind == "evict":
            ev, rep, perm = events["evict"][int(step)]
            kv = dict(f.split("=") for f in fields)
            assert ev[0][0] == int(kv["req"]) and ev[0][4] == int(kv["rows"])
            assert rep.d2h_bytes == int(kv["bytes"])
            if "hbm" in kv:
                assert rep.paper_hbm_bytes == int(kv["hbm"])
            if "perm" in kv:
                assert perm == [int(x) for x in kv["perm"].split(",")]
        elif kind == "move":
            assert events["move"][int(step)] == fields
        elif kind == "total":
            kv = dict(f.split("=") for f in [step] + fields)
            assert res["steps"] == int(kv["steps"]) and res["d2h"] == int(kv["d2h"])
    # no finish / eviction beyond the golden ones (the table lists moves only
    # at t = 7 and 9, so moves elsewhere are not constrained here)
    gold_steps = {(k, s) for k, s, *_ in _parse_golden() if k in ("finish", "evict")}
    for k in ("finish", "evict"):
        for s in events[k]:
            assert (k, str(s)) in gold_steps, (k, s)


def test_c0prime_interior_eviction(oracle_lib):
    # SURVEY.md Appendix B, C0': at t=12 req 1 finishes and req 0 is evicted at
    # batch index 3, with req 2 moved below it (exercises the rows-below term).
    t = s3synth.c0prime_trace()
    seen = {}

    def rec(step, o, rep, perm, ev, fin, adm, pre):
        if step == 12:
            seen.update(ev=ev, fin=list(fin), rep=rep, pre=pre)

    run_oracle(t, L=1, H=2, D=64, R=64, record=rec)
    assert seen["fin"] == [1]
    assert seen["ev"][0][0] == 0 and seen["ev"][0][1] == 3
    pre = seen["pre"]
    assert pre[4][0] == 2                       # req 2 sits below req 0
    assert seen["rep"].paper_hbm_bytes == 2 * pre[4][4] * 512
    assert seen["rep"].moved_bytes == (pre[4][3] + 1) * 512


# ---------------------------------------------------------------------------
# P3 / P4 / P7: detection, p = 0, byte conservation over whole runs
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("policy,p", [("short", 0.3), ("bucket", 0.0)])
def test_eviction_schedule_closed_form(oracle_lib, policy, p):
    t = s3synth.make_trace(300, seed=5, policy=policy, p=p, max_seq_len=256, prompt_max=40)
    res = run_oracle(t, R=1024)
    kvpt = 4 * 1 * 1 * 8
    total = 0
    for r in range(t.n):
        gens = expected_evictions(int(t.cap[r]), int(t.prompt[r]), int(t.out[r]), t.max_seq_len)
        assert res["evict_gens"].get(r, []) == gens          # P3
        c = int(t.cap[r])
        for _ in gens:
            total += c * kvpt
            c = min(2 * c, t.max_seq_len)
    assert res["d2h"] == total                               # P7 (schedule independent)
    assert sum(res["batch_sizes"]) == int(t.out.sum())       # P7 conservation: sum_t B_t = sum O
    assert res["paper_pcie"] == 2 * total
    if p == 0.0:
        assert res["d2h"] == 0 and not res["evictions"]      # P4


@pytest.mark.parametrize("policy", ["oracle", "bucket", "maxlen"])
def test_no_penalty_without_short_predictions(oracle_lib, policy):
    # P4 / PAPER.md:26: predictions never short -> zero evictions, zero D2H.
    t = s3synth.make_trace(200, seed=9, policy=policy, max_seq_len=256, prompt_max=40)
    res = run_oracle(t, R=2048)
    assert res["d2h"] == 0 and res["paper_pcie"] == 0 and res["paper_hbm"] == 0
    assert sum(res["batch_sizes"]) == int(t.out.sum())


# ---------------------------------------------------------------------------
# P5 compaction brute force against a copy-to-fresh-buffer formulation
# ---------------------------------------------------------------------------

def _compaction_case(statuses, rng):
    n = len(statuses)
    L, H, D, M = 1, 1, 8, 64
    prompts = rng.integers(0, 6, n)
    allocs = np.where(np.array(statuses) == oracle.OVERRUN, 1, rng.integers(2, 6, n))
    prompts = np.where(np.array(statuses) == oracle.OVERRUN, np.maximum(prompts, 0), prompts)
    R = int((prompts + allocs).sum()) + int(rng.integers(0, 5))
    o = oracle.Oracle(L, H, D, M, max(R, M))
    o.submit(np.arange(n), prompts, allocs)
    assert len(o.admit()) == n
    q, k, v, _ = o.make_inputs(np.full(n, 1000, np.int32))
    # statuses are given per request; batch order is FFD order
    statuses = [statuses[s[0]] for s in o.batch()]
    eos = np.array([s == oracle.FINISHED for s in statuses], np.uint8)
    o.decode(q, k, v, eos)
    pre = o.batch()
    A0 = o.arena().copy()
    rep, perm, ev, fin = o.evict_compact()
    post = o.batch()
    A1 = o.arena()
    kvpt = 4 * L * H * D
    # expected: a fresh arena built by copying each survivor, in order, to the
    # running sum of kept caps (no in-place memmove)
    exp_off, run_, exp_perm, moved = [], 0, [], 0
    kept = [i for i, s in enumerate(statuses) if s == oracle.RUNNING]
    for i in range(n):
        exp_perm.append(kept.index(i) if i in kept else -1)
    for i in kept:
        exp_off.append(run_)
        if run_ != pre[i][5]:
            moved += pre[i][3] * kvpt
        run_ += pre[i][4]
    assert list(perm) == exp_perm
    assert [s[5] for s in post] == exp_off
    assert rep.tail == run_ and rep.moved_bytes == moved
    for j, i in enumerate(kept):
        ln, off0, off1 = pre[i][3], pre[i][5], post[j][5]
        assert np.array_equal(A1[off1:off1 + ln], A0[off0:off0 + ln])
    ev_idx = [i for i, s in enumerate(statuses) if s == oracle.OVERRUN]
    assert [e[1] for e in ev] == ev_idx
    assert rep.d2h_bytes == sum(pre[i][3] * kvpt for i in ev_idx)
    assert rep.paper_hbm_bytes == sum(2 * kvpt * sum(p[4] for p in pre[i + 1:]) for i in ev_idx)
    for i in ev_idx:
        host = o.host_kv(pre[i][0])
        assert np.array_equal(host, A0[pre[i][5]:pre[i][5] + pre[i][3]])
    first = next((i for i, s in enumerate(statuses) if s != oracle.RUNNING), n)
    assert rep.first_hole == first


def test_compaction_all_patterns_small(oracle_lib):
    rng = np.random.default_rng(0)
    S = [oracle.RUNNING, oracle.FINISHED, oracle.OVERRUN]
    for n in range(1, 6):
        for statuses in itertools.product(S, repeat=n):
            _compaction_case(list(statuses), rng)


def test_compaction_random_b10(oracle_lib):
    rng = np.random.default_rng(1)
    for _ in range(300):
        _compaction_case(list(rng.integers(0, 3, 10)), rng)


def test_single_eviction_matches_paper_closed_form(oracle_lib):
    # P5(iii): one eviction at batch index i; D2H = S_P(x_i), paper_hbm/2 =
    # sum_{j>i} S_P(x_j) (Eq. PAPER.md:15 numerators); resident-row moves <= it.
    rng = np.random.default_rng(2)
    for n in range(1, 9):
        for i in range(n):
            st = [oracle.RUNNING] * n
            st[i] = oracle.OVERRUN
            _compaction_case(st, rng)


# ---------------------------------------------------------------------------
# P6 first-fit decreasing
# ---------------------------------------------------------------------------

def test_ffd_spec_example(oracle_lib):
    # sizes [5,3,3,2], capacity 8 -> admit [5,3]
    adm = oracle.ffd([5, 3, 3, 2], [0, 1, 2, 3], 8)
    assert adm.tolist() == [True, True, False, False]
    # tie rule (R7): equal caps -> lower req first
    adm = oracle.ffd([3, 3], [9, 4], 3)
    assert adm.tolist() == [False, True]
    # SPEC.md:221 exact-fit replacement; SPEC.md:223 admit into just-freed space
    assert oracle.ffd([7], [0], 7).tolist() == [True]
    assert oracle.ffd([], [], 5).tolist() == []


def test_ffd_maximal_exhaustive(oracle_lib):
    # on <= 12 items, no skipped item fits the residual capacity;
    # and the admitted set is the greedy prefix (checked against brute force
    # over all subsets: it is the lexicographically-greedy feasible set).
    rng = np.random.default_rng(7)
    for trial in range(400):
        n = int(rng.integers(1, 13))
        caps = rng.integers(1, 20, n)
        reqs = rng.permutation(n)
        cap_total = int(rng.integers(0, caps.sum() + 2))
        adm = oracle.ffd(caps, reqs, cap_total)
        used = int(caps[adm].sum())
        assert used <= cap_total
        assert all(caps[i] > cap_total - used for i in range(n) if not adm[i])
        # brute force: among all feasible subsets, FFD's set is the one that is
        # lexicographically maximal in the (cap desc, req asc) order
        if n > 10:
            continue
        order = sorted(range(n), key=lambda i: (-caps[i], reqs[i]))
        best = None
        for mask in range(1 << n):
            if sum(caps[order[j]] for j in range(n) if mask >> (n - 1 - j) & 1) <= cap_total:
                best = mask if best is None or mask > best else best
        exp = np.zeros(n, bool)
        for j in range(n):
            if best >> (n - 1 - j) & 1:
                exp[order[j]] = True
        assert np.array_equal(adm, exp)


def test_ffd_multibin(oracle_lib):
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(0, 30))
        caps = rng.integers(1, 30, n)
        reqs = rng.permutation(n)
        G = int(rng.integers(1, 5))
        free = rng.integers(0, 80, G)
        slots = rng.integers(0, 6, G)
        who = oracle.ffd_multibin(caps, reqs, free, slots)
        for r in range(G):
            assert caps[who == r].sum() <= free[r] and (who == r).sum() <= slots[r]
        # no unassigned item fits any bin's residual (with a slot left)
        for i in np.where(who < 0)[0]:
            for r in range(G):
                assert not (caps[i] <= free[r] - caps[who == r].sum() and (who == r).sum() < slots[r])
        if G == 1:
            assert np.array_equal(who == 0, oracle.ffd(caps, reqs, free[0], slots[0]))


def test_doubling_terminates(oracle_lib):
    # at most ceil(log2(max_len)) evictions per request.
    t = s3synth.make_trace(400, seed=4, policy="short", p=0.9, max_seq_len=256, prompt_max=40)
    res = run_oracle(t, R=600)
    assert max(res["evictions"].values()) <= math.ceil(math.log2(256))


def test_max_running_limits_admission(oracle_lib):
    t = s3synth.make_trace(50, seed=3, policy="oracle", max_seq_len=128, prompt_max=20)
    res = run_oracle(t, R=4096, max_running=4)
    assert max(res["batch_sizes"]) <= 4
    assert sum(res["batch_sizes"]) == int(t.out.sum())


# ---------------------------------------------------------------------------
# P9 multi-rank: G oracle instances + an in-memory sum "allreduce"
# ---------------------------------------------------------------------------

def test_multirank_plan_consistency(oracle_lib):
    G = 3
    t = s3synth.make_trace(240, seed=8, policy="short", p=0.2, max_seq_len=128, prompt_max=20)
    ranks = [oracle.Oracle(1, 1, 8, 128, 400, max_running=40) for _ in range(G)]
    for o in ranks:
        o.submit(t.req_id, t.prompt, t.alloc)
    owner = {}
    tokens = 0
    for step in range(10000):
        for o in ranks:
            o.admit_home()
        M = np.zeros((G, 8), np.int64)
        for r, o in enumerate(ranks):
            M[r] = o.counters()
        # every rank holds the identical fresh pool (row 4 equal on all ranks)
        assert len(set(M[:, 4])) == 1
        plans = [o.admit_shared(G, r, M[:, 0], M[:, 2]) for r, o in enumerate(ranks)]
        for r, pl in enumerate(plans):
            for req in pl:
                assert req not in owner
                owner[req] = r
        if all(o.B == 0 for o in ranks) and M[:, 3].sum() == 0 and ranks[0].counters()[4] == 0:
            break
        for o in ranks:
            if o.B == 0:
                continue
            tokens += o.B
            q, k, v, eos = o.make_inputs(t.out)
            o.decode(q, k, v, eos)
            o.evict_compact()
    assert sorted(owner) == list(range(t.n))          # every request admitted once, fresh
    assert tokens == int(t.out.sum())                 # conservation across ranks


def test_attend_generated_matches_state_machine(oracle_lib):
    # P2: the state machine's arena rows are the generator's, so its decode
    # output equals the pure-function attention of (req, pos, l).
    L, H, D = 2, 2, 64
    o = oracle.Oracle(L, H, D, 64, 128)
    o.submit(np.arange(3), [0, 5, 17], [9, 9, 9])
    o.admit()
    q, k, v, eos = o.make_inputs(np.full(3, 100, np.int32))
    pre = o.batch()
    out, _ = o.decode(q, k, v, eos)
    for b, (req, P, gen, ln, cap, off) in enumerate(pre):
        for l in range(L):
            ref = oracle.attend_generated(L, H, D, 64, 1, req, ln, l)
            assert np.array_equal(out[l, b], ref)


@pytest.mark.parametrize("policy,p", [("short", 0.3), ("oracle", 0.0)])
def test_on_demand_compaction_same_schedule(oracle_lib, policy, p):
    # R27: compacting only when the pool is non-empty after the step's
    # evictions changes no admission, eviction or output -- only offsets
    # while the pool is empty -- and never moves more bytes.
    t = s3synth.make_trace(120, seed=19, policy=policy, p=p, max_seq_len=128, prompt_max=20)
    logs = {}
    for pol in (0, 1):
        o = oracle.Oracle(1, 2, 64, 128, 700, compact_policy=pol)
        o.submit(t.req_id, t.prompt, t.alloc)
        ev = [("admit", tuple(o.admit()))]
        outs, moved, holes = [], 0, 0
        while True:
            c = o.counters()
            if o.B == 0 and c[3] + c[4] == 0:
                break
            q, k, v, eos = o.make_inputs(t.out)
            out, st = o.decode(q, k, v, eos)
            outs.append(out.copy())
            rep, perm, e, fin = o.evict_compact()
            moved += rep.moved_bytes
            ev.append(("step", tuple(perm), tuple(x[0] for x in e), tuple(int(f) for f in fin)))
            ev.append(("admit", tuple(o.admit())))
            b = o.batch()
            if b and b[0][5] != 0 or any(b[i][5] + b[i][4] != b[i + 1][5] for i in range(len(b) - 1)):
                holes += 1
        logs[pol] = (ev, outs, moved, holes)
    assert logs[0][0] == logs[1][0]
    assert all(np.array_equal(a, b) for a, b in zip(logs[0][1], logs[1][1]))
    assert logs[1][2] <= logs[0][2]
    assert logs[0][3] == 0            # every-step policy: never a hole after a step
    assert logs[1][3] > 0             # on demand: holes persist in the drain phase


@pytest.mark.parametrize("H,Hkv", [(8, 2), (4, 1), (4, 4)])
def test_gqa_attention_matches_sdpa_with_repeated_kv(oracle_lib, H, Hkv):
    # NEXT-4: grouped-query attention = MHA with each KV head repeated for its
    # H/Hkv query heads (library cross-check, torch SDPA in fp64).
    L, D = 2, 64
    o = oracle.Oracle(L, H, D, 64, 128, Hkv=Hkv)
    o.submit(np.arange(3), [1, 9, 30], [4, 4, 4])
    o.admit()
    q, k, v, eos = o.make_inputs(np.full(3, 100, np.int32))
    assert k.shape == (L, 3, Hkv, D) and q.shape == (L, 3, H, D)
    out, _ = o.decode(q, k, v, eos)
    A = o.arena()
    G = H // Hkv
    for b, (req, P, gen, ln, cap, off) in enumerate(o.batch()):
        for l in range(L):
            K = torch.from_numpy(oracle.bf16_bits_to_f64(A[off:off + ln, l, 0])).permute(1, 0, 2)
            V = torch.from_numpy(oracle.bf16_bits_to_f64(A[off:off + ln, l, 1])).permute(1, 0, 2)
            K = K.repeat_interleave(G, dim=0)
            V = V.repeat_interleave(G, dim=0)
            Q = torch.from_numpy(oracle.bf16_bits_to_f64(q[l, b]))[:, None, :]
            ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V)[:, 0, :].numpy()
            assert np.allclose(out[l, b], ref, rtol=0, atol=1e-12)
    # kvpt shrinks with the KV heads (PAPER.md:111 formula with d_h -> Hkv*D)
    assert o.kvpt == 4 * L * Hkv * D


# ---------------------------------------------------------------------------
# R28 length stop, R26 worst-fit placement, R27 admission-time compaction
# ---------------------------------------------------------------------------

def test_length_stop_without_eos(oracle_lib):
    # R28: with no EOS ever, a request generates until len == max_len and
    # finishes there (SPEC.md:44 P + O <= max_seq_len); on the way its
    # reservation doubles (P3's closed form with O = max_len - P), and the
    # run terminates with sum_t B_t = sum_r (max_len - P_r).
    t = s3synth.make_trace(120, seed=23, policy="short", p=0.5, max_seq_len=64, prompt_max=20)
    never = s3synth.Trace(t.req_id, t.prompt, np.full(t.n, 1 << 30, np.int32), t.alloc, t.max_seq_len)
    res = run_oracle(never, R=600)
    for r in range(t.n):
        O = t.max_seq_len - int(t.prompt[r])
        assert res["evict_gens"].get(r, []) == expected_evictions(int(t.cap[r]), int(t.prompt[r]), O,
                                                                   t.max_seq_len)
    assert len(res["finished_step"]) == t.n
    assert sum(res["batch_sizes"]) == int((t.max_seq_len - t.prompt.astype(np.int64)).sum())


def test_multibin_worst_fit_placement(oracle_lib):
    # R26: an item goes to the rank with the most free rows (ties: lowest
    # rank) -- first fit would fill rank 0 first.
    who = oracle.ffd_multibin([5, 4, 3], [0, 1, 2], [10, 20, 20], [4, 4, 4])
    # free [10, 20, 20]: 5 -> rank 1 (tie, lower rank) -> [10, 15, 20]; 4 -> rank 2 -> [10, 15, 16];
    # 3 -> rank 2 (16 > 15).  First fit would give [1, 1, 0].
    assert list(who) == [1, 2, 2]
    rng = np.random.default_rng(29)
    for _ in range(300):
        n = int(rng.integers(1, 40))
        G = int(rng.integers(2, 9))
        caps = rng.integers(1, 50, n)
        reqs = rng.permutation(n)
        free = rng.integers(0, 200, G)
        slots = np.full(G, 1 << 20)
        who = oracle.ffd_multibin(caps, reqs, free, slots)
        left = free - np.array([caps[who == r].sum() for r in range(G)])
        assert (left >= 0).all()
        # LPT-style balance bound of greedy worst fit: a rank that received an
        # item had the most free rows when its last item arrived, so it ends at
        # most (that item's cap) below the final maximum.  First fit breaks it.
        for r in range(G):
            if (who == r).any():
                order = np.lexsort((reqs[who == r], -caps[who == r]))
                last_cap = caps[who == r][order[-1]]
                assert left[r] >= left.max() - last_cap


def test_on_demand_compaction_late_submit(oracle_lib):
    # R27 at admission: a step with an empty pool leaves holes; a request
    # submitted later must see the every-step free rows (the advisor's case:
    # without the admission-time shift it would be admitted later or not at all).
    # max-length caps (all 128 rows): finishes leave interior holes
    t = s3synth.make_trace(60, seed=31, policy="maxlen", max_seq_len=128, prompt_max=20)
    first, late = np.arange(40), np.arange(40, 60)
    logs = {}
    for pol in (0, 1):
        o = oracle.Oracle(1, 2, 64, 128, 40 * 128 + 100, compact_policy=pol)
        o.submit(t.req_id[first], t.prompt[first], t.alloc[first])
        ev = [tuple(o.admit())]
        views = []
        step = 0
        while True:
            c = o.counters()
            if o.B == 0 and c[3] + c[4] == 0 and step > 40:
                break
            if o.B:
                q, k, v, eos = o.make_inputs(t.out)
                o.decode(q, k, v, eos)
                o.evict_compact()
            if step == 40:      # between the step's evict_compact (empty pool) and the admission
                o.submit(t.req_id[late], t.prompt[late], t.alloc[late])
            waiting = o.counters()[4] > 0
            ev.append(tuple(o.admit()))
            views.append(tuple(o.batch()) if waiting else None)
            step += 1
        logs[pol] = (ev, views, o.moved_at_admit())
    assert logs[0][0] == logs[1][0]          # identical admissions
    # identical layouts after every admission that had requests waiting (holes
    # stay only while nobody could use them)
    assert logs[0][1] == logs[1][1]
    assert logs[1][1][40] is not None
    assert logs[0][2] == 0 and logs[1][2] > 0


def test_attend_rows_matches_sdpa_and_generated(oracle_lib):
    # s3o_attend_rows (for GEMM-fed inputs) is the same attention: torch SDPA
    # in fp64 on random bf16 rows, and equal to attend_generated on generator rows
    rng = np.random.default_rng(3)
    H, Hkv, D, n = 4, 2, 64, 37
    bits = lambda *s: (rng.integers(-128, 128, s).astype(np.float32) / 64).view(np.uint32).__rshift__(16).astype(np.uint16)
    q, K, V = bits(H, D), bits(n, Hkv, D), bits(n, Hkv, D)
    got = oracle.attend_rows(q, K, V)
    Q = torch.from_numpy(oracle.bf16_bits_to_f64(q))[:, None, :]
    Kt = torch.from_numpy(oracle.bf16_bits_to_f64(K)).permute(1, 0, 2).repeat_interleave(H // Hkv, dim=0)
    Vt = torch.from_numpy(oracle.bf16_bits_to_f64(V)).permute(1, 0, 2).repeat_interleave(H // Hkv, dim=0)
    ref = torch.nn.functional.scaled_dot_product_attention(Q, Kt, Vt)[:, 0, :].numpy()
    assert np.allclose(got, ref, rtol=0, atol=1e-12)
    L, M = 2, 64
    rows = np.stack([np.stack([oracle.gen_kv(L, H, D, M, 1, 5, 1, kv, j, Hkv=Hkv) for kv in (0, 1)]) for j in range(10)])
    qg = oracle.gen_q(L, H, D, M, 1, 5, 1, 9)
    assert np.array_equal(oracle.attend_rows(qg, rows[:, 0], rows[:, 1]),
                          oracle.attend_generated(L, H, D, M, 1, 5, 9, 1, Hkv=Hkv))

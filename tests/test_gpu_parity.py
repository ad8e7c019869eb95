"""GPU path vs oracle parity (-m gpu).  Every call goes through the C ABI.

Bar: bit-exact for slots, offsets, permutations,
eviction lists, byte counters, arena rows and evicted host bytes; attention
within 2e-3 relative error per (layer, slot, head):
    max_d |o_gpu - o_ref| / max(max_d |o_ref|, 2^-20) <= 2e-3.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import s3synth

pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2306_06000_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel_err(out_gpu: np.ndarray, ref: np.ndarray) -> float:
    """Max over (l, b, h) of the per-head relative error."""
    if ref.size == 0:
        return 0.0
    num = np.abs(out_gpu - ref).max(axis=-1)
    den = np.maximum(np.abs(ref).max(axis=-1), 2.0**-20)
    return float((num / den).max())


def u16(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def lockstep(trace, L, H, D, R, C=0, S=0, max_running=4096, staging=True, feed_oracle_inputs=False,
             max_steps=100000, check_arena=True, attn_variant=0, compact_mode=0, poison=False,
             compact_policy=0, Hkv=0, host_io=False, chunks=0, device_out=False, staging_mult=1, late=None,
             reserve_sms=0):
    from paper_2306_06000_b200.engine import S3Engine
    eng = S3Engine(L, H, D, trace.max_seq_len, R, max_running, chunk_rows=C, move_chunk_bytes=S,
                   staging_bytes=(None if staging_mult == 1 else staging_mult * trace.max_seq_len * 4 * L * (Hkv or H) * D)
                   if staging else 0, host_store_bytes=64 << 20, attn_variant=attn_variant,
                   compact_mode=compact_mode, compact_policy=compact_policy, num_kv_heads=Hkv,
                   reserve_sms=reserve_sms)
    eng.profile(True)
    orc = oracle.Oracle(L, H, D, trace.max_seq_len, R, max_running=max_running, compact_policy=compact_policy,
                        Hkv=Hkv)
    # late = (step, request indices): those requests are submitted only at that
    # step, between evict_compact and admit (R27's admission-time shift)
    first = np.ones(trace.n, bool)
    if late is not None:
        first[late[1]] = False
    eng.submit(trace.req_id[first], trace.prompt[first], trace.alloc[first], trace.out[first])
    orc.submit(trace.req_id[first], trace.prompt[first], trace.alloc[first])
    _, adm_g = eng.admit()
    adm_o = orc.admit()
    assert adm_g == adm_o
    worst, steps, stats = 0.0, 0, dict(evictions=0, moved=0, splits=0)
    HD = H * D
    KD = (Hkv or H) * D
    if host_io:
        # s3_decode_step_host: pinned host inputs and output
        hq = torch.empty(eng.q.numel(), dtype=torch.bfloat16, pin_memory=True)
        hk = torch.empty(eng.k_new.numel(), dtype=torch.bfloat16, pin_memory=True)
        hv = torch.empty(eng.v_new.numel(), dtype=torch.bfloat16, pin_memory=True)
        he = torch.empty(eng.eos.numel(), dtype=torch.uint8, pin_memory=True)
        ho = torch.empty(eng.out.numel(), dtype=torch.float32, pin_memory=True)
    moved_admit = 0
    while True:
        c = orc.counters()
        if orc.B == 0 and c[3] + c[4] == 0 and (late is None or steps > late[0]):
            assert eng.B == 0
            break
        assert steps < max_steps
        B = orc.B
        assert eng.batch_view() == orc.batch(), f"step {steps}: batch views differ"
        if poison:
            # T5: every arena row that is not resident (slack, free tail, vacated
            # rows) becomes bf16 NaN; a kernel that reads one leaks NaN into out
            resident = torch.zeros(R, dtype=torch.bool)
            for (_, _, _, ln, _, off) in orc.batch():
                resident[off:off + ln] = True
            eng.arena_rows_view()[(~resident).to(eng.device)] = float("nan")
        q, k, v, eos = orc.make_inputs(trace.out)
        n = L * B * HD
        nk = L * B * KD
        if B:
            if feed_oracle_inputs:
                eng.q[:n].copy_(torch.from_numpy(q.reshape(-1).view(np.int16)).view(torch.bfloat16))
                eng.k_new[:nk].copy_(torch.from_numpy(k.reshape(-1).view(np.int16)).view(torch.bfloat16))
                eng.v_new[:nk].copy_(torch.from_numpy(v.reshape(-1).view(np.int16)).view(torch.bfloat16))
                eng.eos[:B].copy_(torch.from_numpy(eos))
            else:
                eng.synth_inputs()
                # T0 at run time: the CUDA generator equals the oracle's
                assert np.array_equal(u16(eng.q[:n]), q.reshape(-1))
                assert np.array_equal(u16(eng.k_new[:nk]), k.reshape(-1))
                assert np.array_equal(u16(eng.v_new[:nk]), v.reshape(-1))
                assert np.array_equal(eng.eos[:B].cpu().numpy(), eos)
        ref, st = orc.decode(q, k, v, eos)
        if host_io:
            if B:
                hq[:n].copy_(eng.q[:n]); hk[:nk].copy_(eng.k_new[:nk]); hv[:nk].copy_(eng.v_new[:nk])
                he[:B].copy_(eng.eos[:B])
                ho[:n].fill_(float("nan"))
                # NaN-poison the landing buffers: a kernel that reads a chunk before
                # its copy landed leaks NaN into out
                eng.q.fill_(float("nan")); eng.k_new.fill_(float("nan")); eng.v_new.fill_(float("nan"))
                eng.out.fill_(float("nan"))
                eng.eos.fill_(0)
            torch.cuda.synchronize()
            eng.decode_host(hq, hk, hv, he, ho, chunks=chunks, device_out=device_out)
            torch.cuda.synchronize()
        else:
            eng.decode()
        if B:
            got = (ho[:n] if host_io else eng.out[:n]).cpu().numpy().reshape(L, B, H, D).astype(np.float64)
            err = rel_err(got, ref)
            worst = max(worst, err)
            assert err <= TOL, f"step {steps}: attention rel err {err}"
        rep_o, perm_o, ev_o, fin_o = orc.evict_compact()
        rep_g, perm_g, ev_g, fin_g = eng.evict_compact()
        for f in ["n_before", "n_finished", "n_evicted", "n_kept", "d2h_bytes", "moved_bytes",
                  "paper_pcie_bytes", "paper_hbm_bytes", "first_hole"]:
            assert getattr(rep_g, f) == getattr(rep_o, f), (steps, f)
        assert rep_g.tail_rows == rep_o.tail
        assert perm_g == list(perm_o)
        assert [int(x) for x in fin_g] == [int(x) for x in fin_o]
        assert [(e.req_id, e.batch_index, e.prompt_len, e.gen_len, e.len, e.cap_rows, e.new_cap_rows)
                for e in ev_g] == [tuple(e) for e in ev_o]
        if ev_g:
            for e in ev_g:                      # per-request wait (each evictee's own D2H event)
                eng.evict_wait_req(e.req_id)
                host_g = u16(eng.host_rows(e.host_off, e.len).reshape(-1))
                assert np.array_equal(host_g, orc.host_kv(e.req_id).reshape(-1))
        stats["evictions"] += rep_o.n_evicted
        stats["moved"] += rep_o.moved_bytes
        if late is not None and steps == late[0]:
            i = late[1]
            eng.submit(trace.req_id[i], trace.prompt[i], trace.alloc[i], trace.out[i])
            orc.submit(trace.req_id[i], trace.prompt[i], trace.alloc[i])
        arep, adm_g = eng.admit()
        moved_admit += arep.moved_bytes
        adm_o = orc.admit()
        assert moved_admit == orc.moved_at_admit()
        assert adm_g == adm_o, f"step {steps}: admissions differ"
        if check_arena:
            A_o = orc.arena()
            A_g = eng.arena_rows_view()
            for (req, P, gen, ln, cap, off) in orc.batch():
                assert np.array_equal(u16(A_g[off:off + ln].reshape(-1)), A_o[off:off + ln].reshape(-1)), \
                    f"step {steps}: arena rows of req {req} differ"
        steps += 1
    assert eng.verify_resident() == 0
    stats["fused_steps"] = eng.profile_get().fused_steps
    stats["moved_at_admit"] = moved_admit
    eng.close()
    return dict(steps=steps, worst=worst, **stats)


@pytest.mark.parametrize("variant,mode", [(0, 0), (0, 1), (1, 1)])
def test_c0_full_run(variant, mode):
    t = s3synth.c0_trace()
    r = lockstep(t, 1, 2, 64, 64, C=4, S=1024, attn_variant=variant, compact_mode=mode)
    assert r["steps"] == 32 and r["evictions"] == 3


def test_c0prime_full_run_oracle_inputs():
    t = s3synth.c0prime_trace()
    r = lockstep(t, 1, 2, 64, 64, C=3, S=1024, feed_oracle_inputs=True)
    assert r["steps"] == 32


def test_c0_sync_eviction_path():
    t = s3synth.c0_trace()
    r = lockstep(t, 1, 2, 64, 64, C=64, S=1024, staging=False)
    assert r["evictions"] == 3


@pytest.mark.parametrize("variant,mode", [(0, 0), (0, 1), (1, 1)])
def test_gptj_heads_reduced_layers_with_evictions(variant, mode):
    # GPT-J head shape (H=16, D=256), 2 layers; small chunks -> many split-K
    # tiles with ragged tails; small move chunks -> overlapping ordered moves.
    t = s3synth.make_trace(60, seed=3, policy="short", p=0.3, max_seq_len=160, prompt_max=40)
    r = lockstep(t, 2, 16, 256, 1200, C=16, S=4096, max_steps=3000, attn_variant=variant, compact_mode=mode)
    assert r["evictions"] > 0 and r["moved"] > 0
    print("worst rel err", r["worst"])


@pytest.mark.parametrize("variant,mode", [(0, 0), (1, 1)])
def test_head_dim_128(variant, mode):
    t = s3synth.make_trace(40, seed=4, policy="short", p=0.2, max_seq_len=96, prompt_max=20)
    lockstep(t, 3, 4, 128, 400, C=8, S=2048, attn_variant=variant, compact_mode=mode)


def test_tiny_slots_dense_moves():
    # many 1-3 row slots and frequent finishes: stage destinations overlap
    # several source units (the middle-unit wait of k_deps), shifts of 1 row
    rng = np.random.default_rng(17)
    n = 120
    P = rng.integers(0, 3, n).astype(np.int32)
    O = rng.integers(1, 6, n).astype(np.int32)
    alloc = np.where(rng.random(n) < 0.3, np.maximum(1, O - 2), O).astype(np.int32)
    t = s3synth.Trace(np.arange(n, dtype=np.int64), P, O, alloc, 64)
    lockstep(t, 2, 4, 64, 96, C=2, S=1024, compact_mode=0)


def test_max_running_limit_and_p0():
    t = s3synth.make_trace(50, seed=7, policy="bucket", max_seq_len=128, prompt_max=20)
    r = lockstep(t, 1, 2, 64, 2000, C=32, S=1024, max_running=8)
    assert r["evictions"] == 0             # P4: no short predictions -> no penalty


def test_gptj_full_shape_long_sequences():
    # Full GPT-J KV shape (L=28, H=16, D=256), a few long prompts: checks the
    # default chunk C=512 split and the full row stride; 2 steps.
    P = np.array([1500, 900, 511, 2, 1200], np.int32)
    O = np.array([30, 40, 2, 50, 60], np.int32)
    t = s3synth.Trace(np.arange(5, dtype=np.int64), P, O, O.copy(), 2048)
    from paper_2306_06000_b200.engine import S3Engine
    L, H, D = 28, 16, 256
    R = 4500
    eng = S3Engine(L, H, D, 2048, R, 64, host_store_bytes=64 << 20)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    for step in range(2):
        slots = eng.batch_view()
        eng.synth_inputs()
        eng.decode()
        B = len(slots)
        out = eng.out[:L * B * H * D].view(L, B, H, D)
        for b, (req, Pb, gen, ln, cap, off) in enumerate(slots):
            for l in (0, 13, 27):
                ref = oracle.attend_generated(L, H, D, 2048, 1, req, ln, l)
                err = rel_err(out[l, b].cpu().numpy().astype(np.float64)[None], ref[None])
                assert err <= TOL, (step, req, l, err)
        eng.evict_compact()
        eng.admit()
    assert eng.verify_resident() == 0
    eng.close()


def test_bench_configuration_sampled():
    """The bench's launch configuration at full size (C1: GPT-J KV, 8192
    requests, ~160 GB arena, default C and S): sampled outputs against the
    oracle's fp64 attention one at a time, resident rows against the
    generator (P2), and the slot-table invariants after every step."""
    from paper_2306_06000_b200.engine import S3Engine
    L, H, D, M = 28, 16, 256, 2048
    kvpt = 4 * L * H * D
    t = s3synth.make_trace(8192, seed=1, policy="short", p=0.3, max_seq_len=M)
    max_running = 8192
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    free_b, _ = torch.cuda.mem_get_info()
    R = int((free_b - max_running * L * H * D * 10 - (4 << 30) - (8 << 30)) // kvpt)
    eng = S3Engine(L, H, D, M, R, max_running, staging_bytes=4 << 30, host_store_bytes=8 << 30)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    rng = np.random.default_rng(0)
    evictions = 0
    for step in range(60):
        slots = eng.batch_view()
        B = len(slots)
        offs = [s[5] for s in slots]
        assert offs == sorted(offs)
        assert all(slots[i][5] + slots[i][4] <= (slots[i + 1][5] if i + 1 < B else R) for i in range(B))
        assert all(s[3] < s[4] for s in slots)          # len < cap before a decode
        eng.synth_inputs()
        eng.decode()
        if step % 8 == 0:
            lens = np.array([s[3] for s in slots])
            pick = set(rng.choice(B, 6, replace=False).tolist()) | {int(lens.argmax()), int(lens.argmin())}
            out = eng.out[:L * B * H * D].view(L, B, H, D)
            for b in sorted(pick):
                req, P, gen, ln, cap, off = slots[b]
                for l in (0, 27):
                    ref = oracle.attend_generated(L, H, D, M, 1, req, ln, l)
                    err = rel_err(out[l, b].cpu().numpy().astype(np.float64)[None], ref[None])
                    assert err <= TOL, (step, req, ln, l, err)
        rep, perm, ev, fin = eng.evict_compact()
        evictions += rep.n_evicted
        eng.admit()
        if step % 10 == 9:
            assert eng.verify_resident() == 0, step
    print("evictions", evictions)
    assert evictions > 0            # the full-size eviction path (staging, D2H, doubling) ran
    eng.close()


def test_bench_configuration_sampled_host_fed():
    """The e2e leg's path at full size: the same C1-sized configuration driven
    through s3_decode_step_host (pinned host q/k_new/v_new/eos, 16 chunks,
    device out + per-chunk D2H); device landing buffers NaN-poisoned before
    every step; sampled outputs from the HOST buffer against the oracle."""
    from paper_2306_06000_b200.engine import S3Engine
    L, H, D, M = 28, 16, 256, 2048
    kvpt = 4 * L * H * D
    t = s3synth.make_trace(8192, seed=2, policy="short", p=0.1, max_seq_len=M)
    max_running = 8192
    import gc
    gc.collect()
    torch.cuda.empty_cache()                       # arenas of earlier tests go back to the device
    free_b, _ = torch.cuda.mem_get_info()
    R = int((free_b - max_running * L * H * D * 10 - (4 << 30) - (8 << 30)) // kvpt)
    eng = S3Engine(L, H, D, M, R, max_running, staging_bytes=4 << 30, host_store_bytes=8 << 30)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    rows = min(max_running, 2 * eng.B + 64)
    n = L * rows * H * D
    hq, hk, hv = (torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(3))
    ho = torch.empty(n, dtype=torch.float32, pin_memory=True)
    he = torch.empty(max_running, dtype=torch.uint8, pin_memory=True)
    rng = np.random.default_rng(1)
    for step in range(24):
        slots = eng.batch_view()
        B = len(slots)
        assert B <= rows
        m = L * B * H * D
        eng.synth_inputs()
        hq[:m].copy_(eng.q[:m]); hk[:m].copy_(eng.k_new[:m]); hv[:m].copy_(eng.v_new[:m]); he[:B].copy_(eng.eos[:B])
        eng.q.fill_(float("nan")); eng.k_new.fill_(float("nan")); eng.v_new.fill_(float("nan"))
        eng.out.fill_(float("nan"))
        torch.cuda.synchronize()
        eng.decode_host(hq, hk, hv, he, ho)
        torch.cuda.synchronize()
        out = ho[:m].view(L, B, H, D)
        assert torch.isfinite(out).all(), step
        if step % 6 == 0:
            lens = np.array([s[3] for s in slots])
            pick = set(rng.choice(B, 6, replace=False).tolist()) | {int(lens.argmax()), int(lens.argmin()), B - 1}
            for b in sorted(pick):
                req, P, gen, ln, cap, off = slots[b]
                for l in (0, 27):
                    ref = oracle.attend_generated(L, H, D, M, 1, req, ln, l)
                    err = rel_err(out[l, b].numpy().astype(np.float64)[None], ref[None])
                    assert err <= TOL, (step, req, ln, l, err)
        eng.evict_compact()
        eng.admit()
    assert eng.verify_resident() == 0
    eng.close()


@pytest.mark.parametrize("H,Hkv,variant", [(4, 0, 0), (8, 2, 2)])
def test_layer_group_calls(H, Hkv, variant):
    """s3_decode_step over layer groups [0,1), [1,3), [3,4): the append and the
    detection happen only with the last group; results equal one full call
    (CUDA-core MHA and the tensor-core grouped-KV kernel)."""
    from paper_2306_06000_b200.engine import S3Engine
    L, D, M, R = 4, 128, 96, 600
    t = s3synth.make_trace(30, seed=12, policy="short", p=0.3, max_seq_len=M, prompt_max=20)
    eng = S3Engine(L, H, D, M, R, 64, chunk_rows=8, move_chunk_bytes=2048, host_store_bytes=16 << 20,
                   num_kv_heads=Hkv, attn_variant=variant)
    orc = oracle.Oracle(L, H, D, M, R, max_running=64, Hkv=Hkv)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    orc.submit(t.req_id, t.prompt, t.alloc)
    assert eng.admit()[1] == orc.admit()
    HD = H * D
    for step in range(40):
        B = orc.B
        if B == 0:
            break
        q, k, v, eos = orc.make_inputs(t.out)
        ref, _ = orc.decode(q, k, v, eos)
        eng.synth_inputs()
        KD = (Hkv or H) * D
        for (l0, nl) in [(0, 1), (1, 2), (3, 1)]:
            o, ok = l0 * B * HD, l0 * B * KD
            eng.decode(l0, nl, q=eng.q[o:], k_new=eng.k_new[ok:], v_new=eng.v_new[ok:], out=eng.out[o:])
        got = eng.out[:L * B * HD].cpu().numpy().reshape(L, B, H, D).astype(np.float64)
        assert rel_err(got, ref) <= TOL
        rg = eng.evict_compact()
        ro = orc.evict_compact()
        assert rg[1] == list(ro[1]) and rg[0].d2h_bytes == ro[0].d2h_bytes
        assert eng.admit()[1] == orc.admit()
        assert eng.batch_view() == orc.batch()
    assert eng.verify_resident() == 0
    eng.close()


def test_abi_error_codes_and_empty_batch():
    from paper_2306_06000_b200 import s3 as abi
    from paper_2306_06000_b200.engine import S3Engine
    eng = S3Engine(1, 2, 64, 64, 64, 8, host_store_bytes=1 << 20)
    # empty batch: a decode step and an evict/compact are legal no-ops
    eng.decode()
    rep, perm, ev, fin = eng.evict_compact()
    assert rep.n_before == 0 and rep.tail_rows == 0 and perm == [] and ev == []
    with pytest.raises(abi.S3Error) as e:          # no decode since the last evict
        eng.evict_compact()
    assert e.value.code == abi.S3_E_STATE
    with pytest.raises(abi.S3Error) as e:          # prompt + alloc > max_seq_len
        eng.submit([0], [60], [10])
    assert e.value.code == abi.S3_E_INVAL
    with pytest.raises(abi.S3Error) as e:          # alloc < 1
        eng.submit([0], [3], [0])
    assert e.value.code == abi.S3_E_INVAL
    eng.submit([0, 1], [3, 4], [5, 6], [9, 9])
    eng.admit()
    with pytest.raises(abi.S3Error) as e:          # layer range
        abi.s3_decode_step(eng.ctx, 0, 2, eng.q, eng.k_new, eng.v_new, eng.eos, eng.out)
    assert e.value.code == abi.S3_E_INVAL
    eng.synth_inputs()
    eng.decode()
    with pytest.raises(abi.S3Error) as e:          # statuses not consumed
        eng.decode()
    assert e.value.code == abi.S3_E_STATE
    with pytest.raises(abi.S3Error) as e:
        eng.admit()
    assert e.value.code == abi.S3_E_STATE
    rep, perm, ev, fin = eng.evict_compact()     # state intact after the errors
    assert rep.n_before == 2
    eng.admit()
    # host-fed step: host buffers must be pinned, landing buffers non-null
    n = eng.q.numel()
    pq = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    pk = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    pv = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    pe = torch.zeros(8, dtype=torch.uint8, pin_memory=True)
    po = torch.empty(n, dtype=torch.float32, pin_memory=True)
    pageable = torch.empty(n, dtype=torch.float32)
    with pytest.raises(abi.S3Error) as e:          # out not pinned
        abi.s3_decode_step_host(eng.ctx, pq, pk, pv, pe, pageable, eng.q, eng.k_new, eng.v_new, eng.eos)
    assert e.value.code == abi.S3_E_INVAL
    with pytest.raises(abi.S3Error) as e:          # device tensor where a host buffer belongs
        abi.s3_decode_step_host(eng.ctx, eng.q, pk, pv, pe, po, eng.q, eng.k_new, eng.v_new, eng.eos)
    assert e.value.code == abi.S3_E_INVAL
    with pytest.raises(abi.S3Error) as e:          # missing landing buffer
        abi.s3_decode_step_host(eng.ctx, pq, pk, pv, pe, po, None, eng.k_new, eng.v_new, eng.eos)
    assert e.value.code == abi.S3_E_INVAL
    with pytest.raises(abi.S3Error) as e:          # negative pipeline depth
        abi.s3_decode_step_host(eng.ctx, pq, pk, pv, pe, po, eng.q, eng.k_new, eng.v_new, eng.eos, chunks=-1)
    assert e.value.code == abi.S3_E_INVAL
    eng.synth_inputs()                             # still usable: a valid host-fed step goes through
    m = eng.L * eng.B * eng.H * eng.D
    pq[:m].copy_(eng.q[:m]); pk[:m].copy_(eng.k_new[:m]); pv[:m].copy_(eng.v_new[:m]); pe[:eng.B].copy_(eng.eos[:eng.B])
    eng.decode_host(pq, pk, pv, pe, po)
    torch.cuda.synchronize()
    assert torch.isfinite(po[:m]).all()
    eng.evict_compact()
    eng.close()


@pytest.mark.parametrize("mode", [0, 1])
def test_nan_poisoned_non_resident_rows(mode):
    t = s3synth.make_trace(50, seed=23, policy="short", p=0.3, max_seq_len=128, prompt_max=24)
    r = lockstep(t, 2, 4, 128, 700, C=8, S=2048, compact_mode=mode, poison=True)
    assert r["evictions"] > 0


def test_zero_length_prompts():
    # P = 0 requests (SPEC.md:43 allows prompt_tokens >= 0): the first decode
    # attends only to its own new row (P1(i) on the GPU path).
    P = np.array([0, 0, 3, 0, 5, 1], np.int32)
    O = np.array([4, 1, 6, 9, 2, 7], np.int32)
    alloc = np.array([2, 1, 6, 9, 2, 3], np.int32)
    t = s3synth.Trace(np.arange(6, dtype=np.int64), P, O, alloc, 64)
    lockstep(t, 2, 4, 64, 64, C=2, S=1024)


def test_model_proxy_runs_per_layer_path():
    """NEXT-2 proxy: random-weight GEMMs around per-layer decode calls; the
    path must stay consistent (finite outputs, token conservation)."""
    from paper_2306_06000_b200.engine import S3Engine
    from paper_2306_06000_b200.model_proxy import GPTJProxy
    t = s3synth.make_trace(40, seed=31, policy="short", p=0.2, max_seq_len=128, prompt_max=16)
    eng = S3Engine(3, 4, 64, 128, 600, 64, chunk_rows=16, host_store_bytes=16 << 20)
    proxy = GPTJProxy(eng, d_ff=1024)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    tokens, done = 0, False
    for _ in range(5000):
        c = eng.counters_local()
        if eng.B == 0 and c[3] + c[4] == 0:
            done = True
            break
        B = proxy.decode_step()
        tokens += B
        if B:
            assert torch.isfinite(eng.out[:B * 256]).all()
        eng.evict_compact()
        eng.admit()
    assert done
    assert tokens == int(t.out.sum())
    eng.close()


@pytest.mark.parametrize("mode", [0, 1])
def test_on_demand_compaction_policy(mode):
    # R27 on the GPU path (fused and separate pass), through the drain phase
    t = s3synth.make_trace(60, seed=41, policy="short", p=0.3, max_seq_len=128, prompt_max=24)
    r = lockstep(t, 2, 16, 256, 900, C=16, S=4096, compact_mode=mode, compact_policy=1, poison=True)
    assert r["evictions"] > 0


@pytest.mark.parametrize("seed", range(12))
def test_randomized_configurations(seed):
    """Property sweep: random shapes, chunk sizes, move chunks, policies,
    compaction modes, kernel variants, staging on/off; full runs in lockstep."""
    rng = np.random.default_rng(1000 + seed)
    D = int(rng.choice([64, 128, 256]))
    H = int(rng.choice([1, 2, 4, 8])) if D < 256 else int(rng.choice([1, 2, 4]))
    Hkv = int(rng.choice([h for h in (1, 2, 4, 8) if h <= H and H % h == 0]))
    L = int(rng.integers(1, 4))
    M = int(rng.choice([64, 96, 160]))
    n = int(rng.integers(10, 50))
    pol = str(rng.choice(["short", "bucket", "oracle", "maxlen"]))
    t = s3synth.make_trace(n, seed=seed, policy=pol, p=0.3, max_seq_len=M, prompt_max=M // 4)
    R = int(M * rng.integers(1, 6))
    variant = int(rng.integers(0, 2))
    if D == 128 and 2 <= H // Hkv <= 16 and rng.random() < 0.5:
        variant = 2                     # tensor cores for grouped KV
    mode = int(rng.integers(0, 2)) if variant == 0 else 1
    r = lockstep(t, L, H, D, R, C=int(rng.choice([2, 5, 16, 64])), S=int(rng.choice([1024, 4096, 32768])),
                 max_running=int(rng.choice([4, 16, 4096])), staging=bool(rng.integers(0, 2)),
                 attn_variant=variant, compact_mode=mode, compact_policy=int(rng.integers(0, 2)),
                 poison=bool(rng.integers(0, 2)), Hkv=Hkv)
    print(seed, dict(L=L, H=H, Hkv=Hkv, D=D, M=M, n=n, pol=pol, R=R, variant=variant), r)


@pytest.mark.parametrize("H,Hkv,D,variant,mode", [(8, 2, 128, 0, 0), (8, 2, 128, 1, 1), (4, 1, 64, 0, 0),
                                                  (16, 4, 256, 0, 1), (32, 8, 128, 0, 0)])
def test_grouped_query_kv(H, Hkv, D, variant, mode):
    """NEXT-4: grouped-query / multi-query KV through the whole path."""
    t = s3synth.make_trace(40, seed=51, policy="short", p=0.3, max_seq_len=128, prompt_max=24)
    r = lockstep(t, 2, H, D, 800, C=8, S=2048, attn_variant=variant, compact_mode=mode, Hkv=Hkv, poison=True)
    assert r["evictions"] > 0


@pytest.mark.parametrize("H,Hkv,C,policy,mode,staging", [
    (8, 2, 512, "short", 0, True), (32, 8, 48, "short", 0, True), (16, 1, 128, "bucket", 0, True),
    (4, 2, 7, "short", 0, True), (8, 2, 64, "short", 1, True), (8, 2, 512, "short", 0, False),
    (12, 4, 40, "short", 0, True), (24, 3, 96, "short", 0, True), (8, 4, 33, "short", 0, True)])
def test_grouped_query_kv_tensor_cores(H, Hkv, C, policy, mode, staging):
    """attn_variant 2: tcgen05/TMEM/TMA kernel for grouped KV (D = 128); C
    small -> split-K units and tile tails; NaN-poisoned slack rows.  mode 0:
    the row shift and the eviction staging are fused into the kernel (TMA
    tensor stores + ragged-tail warp copy; checked row by row against the
    oracle's arena and host copies every step); mode 1: separate k_move
    pass; no staging: evictions fall back to the unfused path."""
    t = s3synth.make_trace(40, seed=53, policy=policy, p=0.3, max_seq_len=320, prompt_max=200)
    r = lockstep(t, 2, H, 128, 1600, C=C, S=2048, attn_variant=2, Hkv=Hkv, poison=True, compact_mode=mode,
                 staging=staging)
    print("worst", r["worst"], "fused", r["fused_steps"], "of", r["steps"], "evictions", r["evictions"])
    if policy == "short":
        assert r["evictions"] > 0
    if mode == 0 and staging:
        assert r["fused_steps"] >= 0.9 * r["steps"]   # unfused only when a step's evictions overflow staging
    if mode == 1:
        assert r["fused_steps"] == 0


@pytest.mark.parametrize("H,Hkv,seed", [(32, 8, 61), (8, 4, 62), (12, 2, 63)])
def test_tensor_core_tail_packing(H, Hkv, seed):
    """Units longer than one 128-row tile: each head's rows past its last full tile
    (<= 64) share a tile with np other heads' tails, those heads' full tiles first in
    the same item (columns of heads a full tile does not belong to stay -inf until
    their own tiles arrive).  Long prompts so most units have full tiles + a tail of
    every size; fused row shift with evictions and NaN-poisoned slack rows."""
    t = s3synth.make_trace(30, seed=seed, policy="short", p=0.3, max_seq_len=640, prompt_max=420)
    r = lockstep(t, 2, H, 128, 6000, C=512, S=4096, attn_variant=2, Hkv=Hkv, poison=True)
    assert r["evictions"] > 0 and r["worst"] <= TOL


@pytest.mark.parametrize("variant,chunks,C,dev_out,mode", [
    (0, 0, 16, False, 0), (0, 64, 0, False, 0), (0, 3, 16, False, 0), (1, 0, 16, False, 1), (2, 0, 16, False, 0),
    (0, 0, 16, True, 0), (0, 5, 8, True, 0), (0, 64, 0, True, 0), (2, 0, 16, True, 0), (0, 0, 16, True, 1),
    (2, 4, 16, False, 1)])
def test_host_fed_decode_step(variant, chunks, C, dev_out, mode):
    """s3_decode_step_host: pinned host q/k_new/v_new/eos in, pinned host out,
    H2D pipelined with the attention kernel through per-chunk ready words
    (TMA variant) or completed before it (other variants); out either stored
    by the kernels over PCIe or (dev_out) copied per finished chunk by a
    stream that waits on the kernel's per-chunk counters, split-K slots after
    k_combine (small C makes many of them); mode 1 = the separate k_move
    row shift instead of the fused one.  Device landing buffers and the
    device out are NaN-poisoned before every step."""
    if variant == 2:
        H, Hkv, D = 8, 2, 128
    else:
        H, Hkv, D = 4, 0, 64
    t = s3synth.make_trace(48, seed=7, policy="short", p=0.3, max_seq_len=256, prompt_max=64)
    r = lockstep(t, 2, H, D, 2048, C=C, host_io=True, chunks=chunks, attn_variant=variant, Hkv=Hkv,
                 device_out=dev_out, compact_mode=mode)
    assert r["steps"] > 20 and r["worst"] <= TOL


@pytest.mark.parametrize("variant,Hkv,D,H", [(0, 0, 64, 4), (2, 2, 128, 8)])
def test_double_buffered_staging_heavy_evictions(variant, Hkv, D, H):
    """Staging large enough for two maximal evictions is used as two halves
    that alternate per step (a step's evictees are staged while the previous
    step's D2H still reads the other half).  Heavy short predictions; every
    evicted host copy, resident row and output checked against the oracle."""
    t = s3synth.make_trace(60, seed=11, policy="short", p=0.6, max_seq_len=192, prompt_max=48)
    r = lockstep(t, 2, H, D, 1200, C=32, attn_variant=variant, Hkv=Hkv, staging_mult=3, poison=True)
    assert r["evictions"] >= 20 and r["fused_steps"] >= 0.9 * r["steps"]


# ---------------------------------------------------------------------------
# round 2: length stop (R28), admission-time compaction (R27), error paths
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("variant,mode", [(0, 0), (0, 1), (1, 1)])
def test_no_eos_length_stop(variant, mode):
    # the sampler never emits EOS: every request runs to max_len, is evicted and
    # doubled on the way, and finishes by the length stop (never len > cap)
    t = s3synth.make_trace(40, seed=13, policy="short", p=0.6, max_seq_len=48, prompt_max=12)
    t.out[:] = 1 << 30
    r = lockstep(t, 2, 4, 64, 300, C=8, S=1024, attn_variant=variant, compact_mode=mode)
    assert r["evictions"] > 0


def test_no_eos_length_stop_tensor_cores():
    t = s3synth.make_trace(40, seed=14, policy="short", p=0.6, max_seq_len=64, prompt_max=12)
    t.out[:] = 1 << 30
    r = lockstep(t, 2, 8, 128, 400, C=16, attn_variant=2, Hkv=2)
    assert r["evictions"] > 0


@pytest.mark.parametrize("variant,mode", [(0, 0), (0, 1), (2, 0)])
def test_on_demand_late_submit(variant, mode):
    # maxlen caps (all equal) -> finishes leave interior holes; the pool empties;
    # 20 requests arrive between a step's evict_compact and its admission
    t = s3synth.make_trace(60, seed=31, policy="maxlen", max_seq_len=128, prompt_max=20)
    Hkv = 2 if variant == 2 else 0
    r = lockstep(t, 2, 8 if variant == 2 else 4, 128 if variant == 2 else 64, 40 * 128 + 100, C=16,
                 attn_variant=variant, compact_mode=mode, compact_policy=1, Hkv=Hkv,
                 late=(40, np.arange(40, 60)))
    assert r["moved_at_admit"] > 0


def test_duplicate_submit_and_host_store_exhaustion():
    from paper_2306_06000_b200 import s3 as abi
    from paper_2306_06000_b200.engine import S3Engine
    t = s3synth.make_trace(30, seed=2, policy="short", p=1.0, max_seq_len=64, prompt_max=8)
    L, H, D = 1, 2, 64
    kvpt = 4 * L * H * D
    # host store for ~1 eviction only: the fused step must not stage more than fits
    eng = S3Engine(L, H, D, 64, 2000, 64, host_store_bytes=64 * kvpt)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    with pytest.raises(abi.S3Error) as e:
        eng.submit(t.req_id[:1], t.prompt[:1], t.alloc[:1], t.out[:1])      # already live
    assert e.value.code == 1
    with pytest.raises(abi.S3Error) as e:
        eng.submit(np.array([100, 100]), np.array([3, 3]), np.array([4, 4]), np.array([4, 4]))
    assert e.value.code == 1
    eng.admit()
    hit = False
    for _ in range(200):
        if not eng.B:
            break
        eng.synth_inputs()
        eng.decode()
        try:
            eng.evict_compact()
        except abi.S3Error as err:
            assert err.code == 2                         # S3_E_NOMEM, context still usable
            hit = True
            break
        eng.evict_wait()
        eng.admit()
    assert hit
    assert eng.B > 0                                     # state unchanged, not poisoned
    with pytest.raises(abi.S3Error) as e:
        eng.evict_compact()
    assert e.value.code == 2
    eng.close()


@pytest.mark.parametrize("variant,mode", [(0, 0), (2, 0), (0, 1)])
def test_large_batch_multi_cta_prep(variant, mode):
    # B > 2048 slots: k_prep runs as several CTAs (totals published per CTA,
    # header partials combined by the last); lockstep against the oracle
    t = s3synth.make_trace(6000, seed=17, policy="short", p=0.2, max_seq_len=48, prompt_max=10)
    Hkv = 1 if variant == 2 else 0
    r = lockstep(t, 1, 2 if variant == 2 else 2, 128 if variant == 2 else 64, int(t.cap.sum()) + 64,
                 C=16, max_running=8192, attn_variant=variant, Hkv=Hkv, check_arena=False, compact_mode=mode)
    assert r["evictions"] > 0 and (r["fused_steps"] > 0) == (mode == 0)

"""C-ABI library checks that need no GPU (-m "not gpu").

* libs3.so loads and exports every function include/s3.h declares;
* the host planning helpers (the scheduler's FFD) agree
  with the oracle's FFD on random instances (bit-exact);
* config validation and workspace sizing;
* world_size-2 gloo run: counters all-reduced over a real process group,
  every rank computes the same multi-bin plan, equal to the oracle's.
"""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2306_06000_b200 import build as s3build
from paper_2306_06000_b200 import s3 as abi


@pytest.fixture(scope="module")
def s3lib():
    s3build.build()
    return abi.lib()


def test_exports_every_header_symbol(s3lib):
    names = abi.header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(s3lib, n)]
    assert not missing, missing
    assert set(abi._SIGS) == set(names)


def test_plan_ffd_matches_oracle(s3lib, oracle_lib):
    rng = np.random.default_rng(5)
    for _ in range(500):
        n = int(rng.integers(0, 40))
        cap = rng.integers(1, 60, n).astype(np.int64)
        req = rng.permutation(n).astype(np.int64) * 3 + 7
        free = int(rng.integers(0, max(1, cap.sum() + 3)))
        mx = int(rng.integers(0, n + 2))
        got = np.zeros(n, np.uint8)
        cnt = abi.s3_plan_ffd(cap, req, free, mx, got)
        want = oracle.ffd(cap, req, free, mx)
        assert np.array_equal(got.astype(bool), want)
        assert cnt == int(want.sum())


def test_plan_ffd_multibin_matches_oracle(s3lib, oracle_lib):
    rng = np.random.default_rng(6)
    for _ in range(500):
        n = int(rng.integers(0, 40))
        G = int(rng.integers(1, 9))
        cap = rng.integers(1, 60, n).astype(np.int64)
        req = rng.permutation(n).astype(np.int64)
        fr = rng.integers(0, 150, G).astype(np.int64)
        sl = rng.integers(0, 8, G).astype(np.int64)
        got = np.zeros(n, np.int32)
        f2, s2 = fr.copy(), sl.copy()
        abi.s3_plan_ffd_multibin(cap, req, f2, s2, got)
        want = oracle.ffd_multibin(cap, req, fr, sl)
        assert np.array_equal(got, want)


def _cfg(**kw):
    c = dict(num_layers=28, num_heads=16, head_dim=256, max_seq_len=2048, arena_rows=300000,
             max_running=4096, chunk_rows=0, move_chunk_bytes=0, device=0, stream=None, rank=0,
             world=1, synth_seed=1)
    c.update(kw)
    return abi.s3_config(**c)


def test_workspace_query_and_validation(s3lib):
    a, w, s, h = abi.s3_workspace_query(_cfg())
    assert a == (300000 + 8) * 458752            # R rows + 8 guard rows (tensor-core 8-row group loads)
    assert s == 2048 * 458752
    assert 0 < w < 2 * 1024**3           # workspace stays small next to the arena
    for bad in [dict(head_dim=96), dict(arena_rows=1000), dict(max_running=0), dict(world=0),
                dict(rank=2, world=2), dict(move_chunk_bytes=100), dict(num_heads=64)]:
        with pytest.raises(abi.S3Error) as e:
            abi.s3_workspace_query(_cfg(**bad))
        assert e.value.code == abi.S3_E_INVAL


def test_gemm_workspace_plans(s3lib):
    # host-side GEMM planning (no device: 148 SMs assumed): the workspace a plan asks
    # for pins its choices -- 32 KB of stream-K counters plus ONE fp32 reduce-add tile
    # per tile (rows x BN x 4 B) when it splits K, nothing when it does not
    cnt = 32768
    # M <= 64: swapped operands, 128 W rows x 64 batch columns per tile; stream-K only
    # when the N / 128 tiles fill at most half the SMs (output / down projections)
    assert abi.s3_gemm_workspace(8, 4096, 4096, epi=2) == cnt + (4096 // 128) * 128 * 64 * 4
    assert abi.s3_gemm_workspace(64, 4096, 16384, epi=2) == cnt + (4096 // 128) * 128 * 64 * 4
    assert abi.s3_gemm_workspace(8, 12288, 4096, seg_cols=4096) == 0        # 96 tiles: data parallel
    assert abi.s3_gemm_workspace(1, 16384, 4096, epi=1) == 0                # 128 tiles
    # M = 161: single-CTA 128 x 128 tiles (2 x 32 of them), stream-K over the SMs
    assert abi.s3_gemm_workspace(161, 4096, 4096, epi=2) == cnt + 2 * 32 * 128 * 128 * 4
    # large M, full waves of CTA-pair tiles: data parallel
    assert abi.s3_gemm_workspace(4096, 4096, 4096, epi=2) == 0
    with pytest.raises(abi.S3Error):
        abi.s3_gemm_workspace(8, 100, 4096)                                # N not a multiple of 128


def test_init_rejects_missing_buffers(s3lib):
    ctx = C.c_void_p()
    bufs = abi.s3_buffers()
    rc = s3lib.s3_kv_init(C.byref(_cfg(arena_rows=4096)), C.byref(bufs), C.byref(ctx))
    assert rc == abi.S3_E_NOMEM and not ctx.value


# ---------------------------------------------------------------------------
# world_size-2 gloo: multi-rank admission plan (host logic of §8(e))
# ---------------------------------------------------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, result_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    import s3synth
    from paper_2306_06000_b200 import s3 as abi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = s3synth.make_trace(160, seed=13, policy="short", p=0.25, max_seq_len=96, prompt_max=16)
    o = oracle.Oracle(1, 1, 8, 96, 300, max_running=30)
    o.submit(t.req_id, t.prompt, t.alloc)
    fresh = {int(r): int(c) for r, c in zip(t.req_id, t.cap)}
    plans, steps, tokens = [], 0, 0
    while True:
        o.admit_home()
        row = torch.from_numpy(o.counters())
        mat = torch.zeros(world, 8, dtype=torch.int64)
        mat[rank] = row
        dist.all_reduce(mat)                     # the per-step counter exchange
        M = mat.numpy()
        # the library's planner on the shared fresh pool
        ids = np.array(sorted(fresh), np.int64)
        caps = np.array([fresh[i] for i in ids], np.int64)
        who = np.zeros(len(ids), np.int32)
        abi.s3_plan_ffd_multibin(caps, ids, M[:, 0].copy(), M[:, 2].copy(), who)
        mine = sorted(int(i) for i, w in zip(ids, who) if w == rank)
        got = sorted(o.admit_shared(world, rank, M[:, 0], M[:, 2]))
        assert mine == got, (steps, mine, got)
        for i, w in zip(ids, who):
            if w >= 0:
                del fresh[int(i)]
        plans.append(hash(tuple(int(w) for w in who)))
        done = torch.tensor([o.B + int(M[:, 3].sum()) + len(fresh)], dtype=torch.int64)
        dist.all_reduce(done)
        if done.item() == 0:
            break
        if o.B:
            tokens += o.B
            q, k, v, eos = o.make_inputs(t.out)
            o.decode(q, k, v, eos)
            o.evict_compact()
        steps += 1
    tok = torch.tensor([tokens], dtype=torch.int64)
    dist.all_reduce(tok)
    allplans = [None] * world
    dist.all_gather_object(allplans, plans)
    result_q.put((rank, allplans[0] == allplans[1], int(tok.item()), int(t.out.sum())))
    dist.destroy_process_group()


def test_gloo_two_ranks_same_plan(s3lib, oracle_lib):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, tok, want in res:
        assert same                      # identical plans on every rank
        assert tok == want               # every token generated once across ranks

"""Multi-rank path on one GPU (-m gpu): two processes share cuda:0, the
counter exchange runs over a gloo process group.  Each rank runs the CUDA
path through the C ABI in lockstep with its own oracle rank; admissions
(home re-admission + multi-bin FFD over the shared fresh pool, DESIGN.md
R26), slot tables, reports and attention must match the oracle's, and the
two ranks together generate every token exactly once."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    import s3synth
    from paper_2306_06000_b200.engine import S3Engine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, H, D, M, R = 2, 16, 256, 128, 900
    t = s3synth.make_trace(90, seed=21, policy="short", p=0.3, max_seq_len=M, prompt_max=24)
    eng = S3Engine(L, H, D, M, R, 24, chunk_rows=16, move_chunk_bytes=4096, device=0, rank=rank, world=world,
                   host_store_bytes=64 << 20)
    orc = oracle.Oracle(L, H, D, M, R, max_running=24)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    orc.submit(t.req_id, t.prompt, t.alloc)

    def exchange(row):
        mat = torch.zeros(world, 8, dtype=torch.int64)
        mat[rank] = torch.from_numpy(row)
        dist.all_reduce(mat)
        return mat.numpy()

    tokens, worst, steps = 0, 0.0, 0
    while True:
        a = eng.admit_home()[1]
        b = orc.admit_home()
        assert a == b, ("home", steps, a, b)
        row_g = eng.counters_local()
        row_o = orc.counters()
        assert np.array_equal(row_g[:5], row_o[:5]), (steps, row_g, row_o)
        M_all = exchange(row_g)
        a = eng.admit_shared(M_all)[1]
        b = orc.admit_shared(world, rank, M_all[:, 0], M_all[:, 2])
        assert a == b, ("shared", steps, a, b)
        assert eng.batch_view() == orc.batch()
        done = torch.tensor([eng.B + int(M_all[:, 3].sum()) + int(row_g[4])], dtype=torch.int64)
        dist.all_reduce(done)
        if done.item() == 0:
            break
        B = orc.B
        tokens += B
        q_, k_, v_, eos = orc.make_inputs(t.out)
        ref, _ = orc.decode(q_, k_, v_, eos)
        if B:
            eng.synth_inputs()
        eng.decode()
        if B:
            n = L * B * H * D
            got = eng.out[:n].cpu().numpy().reshape(L, B, H, D).astype(np.float64)
            err = (np.abs(got - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 2.0**-20)).max()
            worst = max(worst, float(err))
            assert err <= 2e-3
        rg = eng.evict_compact()
        ro = orc.evict_compact()
        assert rg[1] == list(ro[1]) and rg[0].moved_bytes == ro[0].moved_bytes
        assert rg[0].d2h_bytes == ro[0].d2h_bytes
        steps += 1
        assert steps < 5000
    tok = torch.tensor([tokens], dtype=torch.int64)
    dist.all_reduce(tok)
    assert eng.verify_resident() == 0
    q.put((rank, int(tok.item()), int(t.out.sum()), worst, steps))
    eng.close()
    dist.destroy_process_group()


def test_two_ranks_share_gpu_lockstep():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, tok, want, worst, steps in res:
        assert tok == want


def test_bench_torchrun_two_ranks_gloo():
    """bench.py's N > 1 path (torchrun, counters all-reduced every step)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "10", "--warmup", "3", "--dist-backend", "gloo", "--arena-gb", "12",
           "--requests", "1500", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["gpu_launches"] > 0
    assert j["e2e"]["value"] > 0 and j["e2e"]["h2d_bytes_per_step"] > 0   # host-fed C ABI on both ranks
    rb = j["rank_balance"]
    assert len(rb["attn_gb_per_rank"]) == 2 and rb["attn_bytes_max_over_mean"] >= 1.0
    # the whole-run leg serves every request to completion across both ranks: tokens = sum O
    import s3synth
    t = s3synth.make_trace(3000, seed=1, policy="oracle", max_seq_len=2048)
    assert j["wholerun"]["tokens"] == int(t.out.sum())


def test_bench_nccl_exchange_world1():
    """The N > 1 exchange on the one GPU this pool has: --dist-always creates an NCCL
    process group of one rank, every engine binds libs3's own NCCL communicator
    (s3_nccl_get_unique_id on rank 0, broadcast, s3_comm_init), and every step's counter
    all-reduce (s3_exchange_counters: its own stream, reserve_sms left free by the
    attention grid) runs through the multi-rank admission path (s3_admit_home ->
    all-reduce -> s3_admit_shared); a second run uses torch.distributed's all_reduce
    (--exchange torch).  With one bin the shared multi-bin
    FFD admits exactly what s3_admit does, so the schedule -- tokens in the window and
    over the whole run -- equals the plain world-1 run's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base = [os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "10", "--warmup", "3",
            "--arena-gb", "12", "--requests", "1500", "--no-cpu-baseline"]
    port = _free_port()
    runs = {}
    tr = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
          "--master-addr", "127.0.0.1"]
    for name, cmd in (("nccl", [*tr, "--master-port", str(port), *base, "--dist-always"]),
                      ("torch", [*tr, "--master-port", str(_free_port()), *base, "--dist-always", "--exchange", "torch"]),
                      ("plain", [sys.executable, *base])):
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-3000:]
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1
        runs[name] = json.loads(lines[0])
    x = runs["nccl"]["exchange"]
    assert x["backend"].startswith("nccl (libs3 communicator") and x["world"] == 1 and x["exchanges"] >= 13
    assert runs["plain"]["exchange"] is None
    assert runs["torch"]["exchange"]["backend"].startswith("nccl (torch.distributed")
    for name in ("nccl", "torch"):
        assert runs[name]["tokens"] == runs["plain"]["tokens"]
        assert runs[name]["wholerun"]["tokens"] == runs["plain"]["wholerun"]["tokens"]
        assert runs[name]["wholerun"]["steps"] == runs["plain"]["wholerun"]["steps"]


def test_library_nccl_exchange_in_process():
    """libs3's own NCCL communicator without torch.distributed: a one-rank
    communicator (s3_nccl_get_unique_id -> s3_comm_init), every step's counter
    all-reduce by s3_exchange_counters inside the multi-rank admission path; the
    schedule equals the plain world-1 engine's step by step, and s3_counters_get
    reports the last exchanged matrix."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    import s3synth
    from paper_2306_06000_b200 import s3 as abi
    from paper_2306_06000_b200.engine import S3Engine
    t = s3synth.make_trace(60, seed=5, policy="short", p=0.3, max_seq_len=128, prompt_max=24)
    L, H, D, R = 2, 4, 64, 1500
    engs = [S3Engine(L, H, D, 128, R, 32, device=0, host_store_bytes=64 << 20, exchange_admission=x,
                     reserve_sms=4 if x else 0) for x in (False, True)]
    engs[1].comm_init(abi.s3_nccl_get_unique_id())
    for e in engs:
        e.submit(t.req_id, t.prompt, t.alloc, t.out)
        e.initial_admit()
    steps = 0
    while engs[0].B or engs[0].counters_local()[3] + engs[0].counters_local()[4]:
        stats = [e.step() for e in engs]
        assert stats[0] == stats[1], (steps, stats)
        assert engs[0].batch_view() == engs[1].batch_view()
        steps += 1
        assert steps < 2000
    c = engs[1].counters_get()
    row = engs[1].counters_local()
    assert c.world == 1 and c.exchanges == steps + 1
    assert c.rank_free_rows[0] == row[0] and c.tokens_total == row[7] == int(t.out.sum())
    for e in engs:
        e.close()

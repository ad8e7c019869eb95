"""Overlap evidence on one B200 (-m gpu).

* reserve_sms: the persistent attention grid leaves SMs free, so a kernel on
  another stream -- the multi-GPU counter all-reduce -- runs
  DURING the attention pass.  Stand-in: a one-CTA kernel with 100 KB of
  dynamic shared memory (it cannot share an SM with the attention kernel).
  With the default multi-GPU reservation it finishes early in the pass; with
  no reservation it waits for the pass to drain (the control).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import tempfile

import numpy as np
import pytest
import torch

import s3synth

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def probe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2306_06000_b200 import build
    build.build()
    so = os.path.join(tempfile.mkdtemp(), "libprobe.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "probe", "probe.cu")])
    lib = C.CDLL(so)
    lib.probe_launch.argtypes = [C.c_void_p, C.c_int, C.c_longlong, C.c_void_p]
    lib.probe_launch.restype = C.c_int
    return lib


def _attention_vs_probe(probe, reserve_sms):
    from paper_2306_06000_b200.engine import S3Engine
    L, H, D = 4, 16, 256
    t = s3synth.make_trace(240, seed=3, policy="oracle", max_seq_len=2048)
    t.prompt[:] = 1200                                  # long contexts: a pass of ~15 GB
    t.alloc[:] = np.minimum(t.alloc, 2048 - 1200)
    t.out[:] = np.minimum(t.out, t.alloc)
    R = int((t.prompt.astype(np.int64) + t.alloc).sum()) + 16
    eng = S3Engine(L, H, D, 2048, R, 256, device=0, host_store_bytes=1 << 26, reserve_sms=reserve_sms)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    side = torch.cuda.Stream()
    ts = torch.zeros(2, dtype=torch.int64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    res = []
    # warm-up: module load and attribute setting of the probe happen on its first launch
    assert probe.probe_launch(C.c_void_p(side.cuda_stream), 100 * 1024, 1000, C.c_void_p(ts.data_ptr())) == 0
    torch.cuda.synchronize()
    for _ in range(4):                                   # the first step also warms launch configurations
        eng.synth_inputs()
        torch.cuda.synchronize()
        ev[0].record()
        eng.decode()
        ev[1].record()
        side.wait_event(ev[0])
        rc = probe.probe_launch(C.c_void_p(side.cuda_stream), 100 * 1024, 20000, C.c_void_p(ts.data_ptr()))
        assert rc == 0
        ev[2].record(side)
        torch.cuda.synchronize()
        attn = ev[0].elapsed_time(ev[1])
        done = ev[0].elapsed_time(ev[2])
        res.append((attn, done))
        eng.evict_compact()
        eng.admit()
    eng.close()
    return res[1:]


def test_reserved_sms_let_a_side_stream_kernel_run_during_attention(probe):
    if os.environ.get("CUDA_INJECTION64_PATH"):
        pytest.skip("timing evidence is meaningless under compute-sanitizer")
    with_res = _attention_vs_probe(probe, 4)
    without = _attention_vs_probe(probe, -1)
    print("attention ms, probe done ms (reserve 4):", with_res, " (none):", without)
    for attn, done in with_res:
        assert attn > 1.0 and done < 0.3 * attn
    for attn, done in without:                          # control: it queues behind the pass
        assert done > 0.7 * attn


def test_eviction_d2h_overlaps_attention():
    """Per-evictee staged-row counters: each evictee's D2H starts as soon as the
    fused attention pass has staged its rows, not after the pass (PAPER.md:174
    "asynchronously").  GPT-J-shaped rows, short(0.9) mispredictions."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if os.environ.get("CUDA_INJECTION64_PATH"):
        pytest.skip("timing evidence is meaningless under compute-sanitizer")
    from paper_2306_06000_b200.engine import S3Engine
    # 90 % short predictions: ~43 evictions in steps 5..104 (length-only oracle replay)
    t = s3synth.make_trace(3000, seed=7, policy="short", p=0.9, max_seq_len=2048)
    L, H, D = 28, 16, 256
    R = 60000                                           # ~27.5 GB of GPT-J KV rows
    eng = S3Engine(L, H, D, 2048, R, 4096, device=0, staging_bytes=4 << 30, host_store_bytes=8 << 30)
    eng.submit(t.req_id, t.prompt, t.alloc, t.out)
    eng.admit()
    for _ in range(5):
        eng.step()
    eng.profile(True)
    ev = stage = 0
    for _ in range(100):
        s = eng.step()
        ev += s.evicted
        stage += s.stage_reload_bytes
    prof = eng.profile_get()
    eng.close()
    frac = prof.d2h_overlap_ms / prof.d2h_ms
    print(f"evictions {ev}, d2h {prof.d2h_bytes / 1e9:.2f} GB in {prof.d2h_ms:.2f} ms, overlap {frac:.3f}, "
          f"reloaded from staging {stage / 1e9:.2f} GB")
    assert ev >= 10 and prof.d2h_copies >= ev
    # A copy that waits for the end of the pass (round 1) overlaps nothing (0.0 here).  The
    # evictees of this small pool sit near the arena's tail (recent admissions with short
    # reservations), so they are staged in the last part of the pass and each 0.3 ms copy
    # outlasts it: measured 0.50-0.6 on B200 (the deep C2 bench leg, 0.98).
    assert frac >= 0.3

"""Seeded synthetic inputs shared by the oracle tests and the CUDA harness.

This module holds NONE of the method's arithmetic (no attention, no scan, no
compaction, no FFD).  It only produces inputs:

* request traces (prompt length P, actual output length O) with the
  "Alpaca-like" length mix of SURVEY.md §8(d) / DESIGN.md "Input recipe";
* the synthetic length predictor's allocations (policies ``oracle``,
  ``bucket``, ``maxlen``, ``short(p)``) that stand in for the paper's
  DistilBERT bucket classifier (PAPER.md:155-161 [§3 Predictor], replaced
  because it needs trained weights);
* the toy traces C0 / C0' of SURVEY.md Appendix B;
* a numpy reference of the counter-based KV / q value generator
  (DESIGN.md "Synthetic data contract").  The oracle (C) and the CUDA path
  each implement the same generator independently; this numpy copy exists so
  the tests can pin both against a third, independent implementation.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Trace", "make_trace", "c0_trace", "c0prime_trace", "bucket_width",
    "splitmix64", "gen_bytes", "kv_elements", "q_elements",
    "GPTJ", "C0_SHAPE",
]

# Model shapes (L, H, D).  GPT-J-6B: 28 layers, 16 heads x 256 = 4096 model
# dim (reading R3: Table 1's "5120" is a garble).
GPTJ = dict(num_layers=28, num_heads=16, head_dim=256, max_seq_len=2048)
C0_SHAPE = dict(num_layers=1, num_heads=2, head_dim=64, max_seq_len=64)

_M64 = (1 << 64) - 1


@dataclass
class Trace:
    """A request pool.  Arrays are aligned by request id (0..n-1)."""
    req_id: np.ndarray   # int64
    prompt: np.ndarray   # int32, P
    out: np.ndarray      # int32, O (actual output length; only the sampler knows it)
    alloc: np.ndarray    # int32, predicted output allocation (cap = P + alloc)
    max_seq_len: int

    @property
    def n(self) -> int:
        return int(self.req_id.shape[0])

    @property
    def cap(self) -> np.ndarray:
        return (self.prompt.astype(np.int64) + self.alloc).astype(np.int64)


def bucket_width(max_seq_len: int, num_buckets: int = 10) -> int:
    """ceil(max/num_buckets) (reading R17)."""
    return -(-max_seq_len // num_buckets)


def _alloc_for_policy(policy: str, P: np.ndarray, O: np.ndarray, max_len: int,
                      rng: np.random.Generator, p: float) -> np.ndarray:
    w = bucket_width(max_len)
    bucket = np.minimum(w * (np.minimum(O // w, 9) + 1), max_len - P)
    if policy == "oracle":
        return O.copy()
    if policy == "bucket":
        return bucket
    if policy == "maxlen":
        return max_len - P
    if policy == "short":
        u_short = rng.random(O.shape[0])
        u_frac = rng.uniform(0.3, 0.9, O.shape[0])
        short = np.maximum(1, np.floor(O * u_frac).astype(np.int64))
        return np.where(u_short < p, short, bucket)
    raise ValueError(f"unknown policy {policy!r}")


def make_trace(n: int, seed: int = 1, policy: str = "oracle", p: float = 0.0,
               max_seq_len: int = 2048, prompt_max: int = 512) -> Trace:
    """Alpaca-like trace.

    P ~ round(LogNormal(ln 20 - 0.18, 0.6)) clipped to [1, prompt_max];
    O ~ round(LogNormal(ln 100 - 0.245, 0.7)) clipped to [1, max_len - P].
    Means: E[P] ~= 20, E[O] ~= 100.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    P = np.rint(rng.lognormal(math.log(20.0) - 0.18, 0.6, n)).astype(np.int64)
    P = np.clip(P, 1, min(prompt_max, max_seq_len - 1))
    O = np.rint(rng.lognormal(math.log(100.0) - 0.245, 0.7, n)).astype(np.int64)
    O = np.clip(O, 1, max_seq_len - P)
    alloc = _alloc_for_policy(policy, P, O, max_seq_len, rng, p)
    return Trace(req_id=np.arange(n, dtype=np.int64), prompt=P.astype(np.int32),
                 out=O.astype(np.int32), alloc=alloc.astype(np.int32),
                 max_seq_len=max_seq_len)


def c0_trace() -> Trace:
    """SURVEY.md Appendix B toy pool: 8 requests, two short mispredictions."""
    P = np.array([4, 6, 3, 5, 2, 7, 4, 3], dtype=np.int32)
    O = np.array([10, 5, 20, 8, 14, 6, 12, 9], dtype=np.int32)
    alloc = O.copy()
    alloc[2] = 8
    alloc[4] = 6
    return Trace(np.arange(8, dtype=np.int64), P, O, alloc, 64)


def c0prime_trace() -> Trace:
    """Appendix B variant C0': alloc0 = 5, alloc4 = O4 = 14 (interior eviction)."""
    t = c0_trace()
    t.alloc[0] = 5
    t.alloc[4] = 14
    return t


# ---------------------------------------------------------------------------
# Counter-based value generator (numpy reference copy).
#
#   splitmix64(x): z = x + 0x9E3779B97F4A7C15
#                  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
#                  z = (z ^ (z >> 27)) * 0x94D049BB133111EB
#                  return z ^ (z >> 31)            (uint64, wrapping)
#   g(req,l,kv,pos,h,d8) = ((((req*L + l)*2 + kv)*MAXLEN + pos)*H + h)*(D/8) + d8
#   z = splitmix64(seed ^ (tag << 60) ^ g)   tag 0 = KV rows, tag 1 = q (kv = 0)
#   element d = 8*d8 + j takes byte j of z:  k8 = ((z >> 8j) & 0xFF) - 128
#   KV element = k8 / 128,  q element = k8 / 32      (both exact in bf16)
# ---------------------------------------------------------------------------

def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def gen_bytes(seed: int, tag: int, req, l, kv, pos, L: int, H: int, D: int,
              max_len: int) -> np.ndarray:
    """int8-valued k8 for all (h, d) of one (req, l, kv, pos): shape [H, D]."""
    g = ((((np.uint64(req) * np.uint64(L) + np.uint64(l)) * np.uint64(2) + np.uint64(kv))
          * np.uint64(max_len) + np.uint64(pos)) * np.uint64(H))
    h = np.arange(H, dtype=np.uint64)[:, None]
    d8 = np.arange(D // 8, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        idx = (g + h) * np.uint64(D // 8) + d8
    x = np.uint64(seed) ^ (np.uint64(tag) << np.uint64(60)) ^ idx
    z = splitmix64(x)                                      # [H, D/8]
    shifts = (np.arange(8, dtype=np.uint64) * np.uint64(8))
    b = ((z[:, :, None] >> shifts[None, None, :]) & np.uint64(0xFF)).astype(np.int32)
    return (b - 128).reshape(H, D)


def kv_elements(seed, req, l, kv, pos, L, H, D, max_len) -> np.ndarray:
    """KV element values (float64, exactly representable in bf16): [H, D]."""
    return gen_bytes(seed, 0, req, l, kv, pos, L, H, D, max_len) / 128.0


def q_elements(seed, req, l, pos, L, H, D, max_len) -> np.ndarray:
    """q element values (float64, exactly representable in bf16): [H, D]."""
    return gen_bytes(seed, 1, req, l, 0, pos, L, H, D, max_len) / 32.0

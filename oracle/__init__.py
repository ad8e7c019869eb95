"""TEST INFRASTRUCTURE ONLY: ctypes loader for the plain-C S^3 oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2306_06000_b200``) never imports it and shares no code
with it.  See ``oracle/s3_oracle.c`` for the citations of each step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "s3_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_s3.so")

RUNNING, FINISHED, OVERRUN = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2; -fopenmp only for the optional
    thread split of the attention loop, off unless set_threads(n > 1))."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "s3_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Config(C.Structure):
    _fields_ = [("L", C.c_int32), ("H", C.c_int32), ("D", C.c_int32), ("max_len", C.c_int32),
                ("R", C.c_int64), ("max_running", C.c_int32), ("seed", C.c_uint64),
                ("compact_policy", C.c_int32), ("Hkv", C.c_int32)]


class Slot(C.Structure):
    _fields_ = [("req", C.c_int64), ("prompt", C.c_int32), ("gen", C.c_int32),
                ("len", C.c_int32), ("cap", C.c_int32), ("off", C.c_int64)]


class Evicted(C.Structure):
    _fields_ = [("req", C.c_int64), ("batch_index", C.c_int32), ("prompt", C.c_int32),
                ("gen", C.c_int32), ("len", C.c_int32), ("cap", C.c_int32), ("new_cap", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("n_before", C.c_int32), ("n_finished", C.c_int32), ("n_evicted", C.c_int32),
                ("n_kept", C.c_int32), ("tail", C.c_int64), ("d2h_bytes", C.c_int64),
                ("moved_bytes", C.c_int64), ("paper_pcie_bytes", C.c_int64),
                ("paper_hbm_bytes", C.c_int64), ("first_hole", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
        sig = {
            "s3o_kv_bytes_per_token": (i64, [i64, i64, i64]),
            "s3o_eviction_penalty": (f64, [f64, f64, f64, f64]),
            "s3o_pool_penalty": (f64, [f64, f64, f64, f64, f64, f64]),
            "s3o_underutilization_ratio": (f64, [i64, P, P]),
            "s3o_splitmix64": (C.c_uint64, [C.c_uint64]),
            "s3o_gen_kv": (None, [P, i64, i32, i32, i32, P]),
            "s3o_gen_q": (None, [P, i64, i32, i32, P]),
            "s3o_ffd": (i32, [i32, P, P, i64, i32, P]),
            "s3o_ffd_multibin": (i32, [i32, P, P, i32, P, P, P]),
            "s3o_create": (P, [P]),
            "s3o_destroy": (None, [P]),
            "s3o_submit": (C.c_int, [P, i32, P, P, P]),
            "s3o_batch": (i32, [P, P]),
            "s3o_arena": (P, [P]),
            "s3o_host_kv": (i64, [P, i64, P]),
            "s3o_make_inputs": (None, [P, P, P, P, P, P]),
            "s3o_decode": (C.c_int, [P, P, P, P, P, P, P]),
            "s3o_set_threads": (None, [C.c_int]),
            "s3o_evict_compact": (C.c_int, [P, P, P, P, P]),
            "s3o_admit": (i32, [P, P]),
            "s3o_admit_home": (i32, [P, P]),
            "s3o_admit_shared": (i32, [P, i32, i32, P, P, P]),
            "s3o_counters": (None, [P, P]),
            "s3o_moved_at_admit": (i64, [P]),
            "s3o_attend_generated": (None, [P, i64, i32, i32, P]),
            "s3o_attend_rows": (None, [P, P, P, i64, i32, i32, i32, i32, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---- closed forms -------------------------------------------------------

def kv_bytes_per_token(L, H, D) -> int:
    return int(lib().s3o_kv_bytes_per_token(L, H, D))


def eviction_penalty(sp_i, sum_below, bw_h2d, bw_hbm) -> float:
    return float(lib().s3o_eviction_penalty(sp_i, sum_below, bw_h2d, bw_hbm))


def pool_penalty(p, N, sp_mean, sum_resident, bw_h2d, bw_hbm) -> float:
    return float(lib().s3o_pool_penalty(p, N, sp_mean, sum_resident, bw_h2d, bw_hbm))


def underutilization_ratio(s_actual, s_pred) -> float:
    a = np.ascontiguousarray(s_actual, dtype=np.int64)
    p = np.ascontiguousarray(s_pred, dtype=np.int64)
    return float(lib().s3o_underutilization_ratio(a.shape[0], _p(a), _p(p)))


def ffd(caps, reqs, free_rows, max_items=1 << 30) -> np.ndarray:
    cap = np.ascontiguousarray(caps, dtype=np.int64)
    req = np.ascontiguousarray(reqs, dtype=np.int64)
    adm = np.zeros(cap.shape[0], dtype=np.uint8)
    lib().s3o_ffd(cap.shape[0], _p(cap), _p(req), int(free_rows), int(max_items), _p(adm))
    return adm.astype(bool)


def ffd_multibin(caps, reqs, free_by_rank, slots_by_rank) -> np.ndarray:
    cap = np.ascontiguousarray(caps, dtype=np.int64)
    req = np.ascontiguousarray(reqs, dtype=np.int64)
    fr = np.ascontiguousarray(free_by_rank, dtype=np.int64).copy()
    sl = np.ascontiguousarray(slots_by_rank, dtype=np.int64).copy()
    who = np.zeros(cap.shape[0], dtype=np.int32)
    lib().s3o_ffd_multibin(cap.shape[0], _p(cap), _p(req), fr.shape[0], _p(fr), _p(sl), _p(who))
    return who


def gen_kv(L, H, D, max_len, seed, req, l, kv, pos, Hkv=0) -> np.ndarray:
    cfg = Config(L, H, D, max_len, max_len, 1, seed, 0, Hkv)
    nh = Hkv or H
    out = np.zeros(nh * D, dtype=np.uint16)
    lib().s3o_gen_kv(C.byref(cfg), req, l, kv, pos, _p(out))
    return out.reshape(nh, D)


def gen_q(L, H, D, max_len, seed, req, l, pos) -> np.ndarray:
    cfg = Config(L, H, D, max_len, max_len, 1, seed, 0, 0)
    out = np.zeros(H * D, dtype=np.uint16)
    lib().s3o_gen_q(C.byref(cfg), req, l, pos, _p(out))
    return out.reshape(H, D)


def attend_generated(L, H, D, max_len, seed, req, pos, l, Hkv=0) -> np.ndarray:
    """fp64 attention of request req at position pos, layer l, when its rows
    are the generator's (see s3o_attend_generated)."""
    cfg = Config(L, H, D, max_len, max_len, 1, seed, 0, Hkv)
    out = np.zeros(H * D, dtype=np.float64)
    lib().s3o_attend_generated(C.byref(cfg), req, pos, l, _p(out))
    return out.reshape(H, D)


def set_threads(n: int) -> None:
    """Threads of the oracle's attention loop (1 = the plain sequential oracle)."""
    lib().s3o_set_threads(int(n))


def attend_rows(q, K, V):
    """fp64 attention of one layer's query heads q [H][D] (bf16 bits) over the
    rows K, V [n][Hkv][D] (bf16 bits); returns [H][D]."""
    q = np.ascontiguousarray(q, dtype=np.uint16)
    K = np.ascontiguousarray(K, dtype=np.uint16)
    V = np.ascontiguousarray(V, dtype=np.uint16)
    n, Hkv, D = K.shape
    H = q.shape[0]
    out = np.zeros(H * D, dtype=np.float64)
    lib().s3o_attend_rows(_p(q), _p(K), _p(V), Hkv * D, n, H, Hkv, D, _p(out))
    return out.reshape(H, D)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


class Oracle:
    """The oracle state machine (one per simulated rank)."""

    def __init__(self, L, H, D, max_len, R, max_running=1 << 20, seed=1, compact_policy=0, Hkv=0):
        self.L, self.H, self.D, self.max_len, self.R = L, H, D, max_len, R
        self.Hkv = Hkv or H
        self.seed = seed
        self.max_running = max_running
        self.cfg = Config(L, H, D, max_len, R, max_running, seed, compact_policy, Hkv)
        self.h = lib().s3o_create(C.byref(self.cfg))
        if not self.h:
            raise ValueError("invalid oracle config")
        self.row_elems = 2 * L * self.Hkv * D
        self.kvpt = 4 * L * self.Hkv * D
        self.n_submitted = 0

    def __del__(self):
        if getattr(self, "h", None):
            lib().s3o_destroy(self.h)
            self.h = None

    def submit(self, req, prompt, alloc):
        req = np.ascontiguousarray(req, dtype=np.int64)
        prompt = np.ascontiguousarray(prompt, dtype=np.int32)
        alloc = np.ascontiguousarray(alloc, dtype=np.int32)
        rc = lib().s3o_submit(self.h, req.shape[0], _p(req), _p(prompt), _p(alloc))
        if rc:
            raise ValueError("invalid request")
        self.n_submitted += int(req.shape[0])

    def batch(self):
        B = lib().s3o_batch(self.h, None)
        arr = (Slot * max(B, 1))()
        lib().s3o_batch(self.h, C.cast(arr, C.c_void_p))
        return [(s.req, s.prompt, s.gen, s.len, s.cap, s.off) for s in arr[:B]]

    @property
    def B(self) -> int:
        return int(lib().s3o_batch(self.h, None))

    def arena(self) -> np.ndarray:
        ptr = lib().s3o_arena(self.h)
        n = self.R * self.row_elems
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint16)), shape=(n,)).reshape(
            self.R, self.L, 2, self.Hkv, self.D)

    def host_kv(self, req):
        ptr = C.c_void_p()
        rows = lib().s3o_host_kv(self.h, req, C.byref(ptr))
        if rows < 0:
            return None
        n = rows * self.row_elems
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint16)), shape=(n,)).reshape(
            rows, self.L, 2, self.Hkv, self.D).copy()

    def make_inputs(self, out_len_by_req):
        B = self.B
        n = self.L * B * self.H * self.D
        nk = self.L * B * self.Hkv * self.D
        q = np.zeros(max(n, 1), np.uint16)
        k = np.zeros(max(nk, 1), np.uint16)
        v = np.zeros(max(nk, 1), np.uint16)
        eos = np.zeros(max(B, 1), np.uint8)
        o = np.ascontiguousarray(out_len_by_req, dtype=np.int32)
        lib().s3o_make_inputs(self.h, _p(o), _p(q), _p(k), _p(v), _p(eos))
        return (q[:n].reshape(self.L, B, self.H, self.D), k[:nk].reshape(self.L, B, self.Hkv, self.D),
                v[:nk].reshape(self.L, B, self.Hkv, self.D), eos[:B])

    def decode(self, q, k, v, eos):
        B = self.B
        out = np.zeros(max(self.L * B * self.H * self.D, 1), np.float64)
        st = np.zeros(max(B, 1), np.uint8)
        q = np.ascontiguousarray(q, dtype=np.uint16)
        k = np.ascontiguousarray(k, dtype=np.uint16)
        v = np.ascontiguousarray(v, dtype=np.uint16)
        eos = np.ascontiguousarray(eos, dtype=np.uint8)
        rc = lib().s3o_decode(self.h, _p(q), _p(k), _p(v), _p(eos), _p(out), _p(st))
        if rc:
            raise RuntimeError(f"oracle decode failed rc={rc}")
        return out[: self.L * B * self.H * self.D].reshape(self.L, B, self.H, self.D), st[:B]

    def evict_compact(self):
        B = max(self.B, 1)
        rep = Report()
        perm = np.zeros(B, np.int32)
        ev = (Evicted * B)()
        fin = np.zeros(B, np.int64)
        rc = lib().s3o_evict_compact(self.h, C.byref(rep), _p(perm), C.cast(ev, C.c_void_p), _p(fin))
        if rc:
            raise RuntimeError(f"oracle evict_compact failed rc={rc}")
        evicted = [(e.req, e.batch_index, e.prompt, e.gen, e.len, e.cap, e.new_cap)
                   for e in ev[: rep.n_evicted]]
        return rep, perm[: rep.n_before], evicted, fin[: rep.n_finished]

    def _admit_call(self, fn, *args):
        out = np.zeros(self.max_running_cap(), np.int64)
        n = fn(self.h, *args, _p(out))
        if n < 0:
            raise RuntimeError(f"oracle admit failed rc={n}")
        return out[:n].tolist()

    def max_running_cap(self):
        return max(1, self.n_submitted)

    def admit(self):
        return self._admit_call(lib().s3o_admit)

    def admit_home(self):
        return self._admit_call(lib().s3o_admit_home)

    def admit_shared(self, world, rank, free_by_rank, slots_by_rank):
        fr = np.ascontiguousarray(free_by_rank, dtype=np.int64)
        sl = np.ascontiguousarray(slots_by_rank, dtype=np.int64)
        return self._admit_call(lib().s3o_admit_shared, world, rank, _p(fr), _p(sl))

    def moved_at_admit(self) -> int:
        """Bytes shifted by R27's admission-time compactions (on-demand policy)."""
        return int(lib().s3o_moved_at_admit(self.h))

    def counters(self) -> np.ndarray:
        row = np.zeros(8, np.int64)
        lib().s3o_counters(self.h, _p(row))
        return row

"""Thin ctypes binding of include/s3.h (argument marshalling only).

Every function below has the same name as its C entry point and only
converts arguments: torch tensors -> device pointers, numpy / ctypes
structures <-> C structs.  All computation happens in libs3.so.  There is no
fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("S3_LIB") or os.path.join(HERE, "lib", "libs3.so")   # S3_LIB: A/B builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "s3.h")

S3_OK, S3_E_INVAL, S3_E_NOMEM, S3_E_CUDA, S3_E_NCCL, S3_E_STATE, S3_E_UNSCHEDULABLE = 0, 1, 2, 3, 4, 5, 6
S3_RUNNING, S3_FINISHED, S3_OVERRUN = 0, 1, 2
S3_NCOUNTERS = 8
S3_NCCL_ID_BYTES = 128
S3_MAX_RANKS = 64
_NAMES = {0: "S3_OK", 1: "S3_E_INVAL", 2: "S3_E_NOMEM", 3: "S3_E_CUDA", 4: "S3_E_NCCL", 5: "S3_E_STATE",
          6: "S3_E_UNSCHEDULABLE"}


class S3Error(RuntimeError):
    def __init__(self, code: int, where: str, msg: str = ""):
        self.code = code
        super().__init__(f"{where}: {_NAMES.get(code, code)} {msg}")


class s3_config(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_heads", C.c_int32), ("head_dim", C.c_int32),
                ("max_seq_len", C.c_int32), ("arena_rows", C.c_int64), ("max_running", C.c_int32),
                ("chunk_rows", C.c_int32), ("move_chunk_bytes", C.c_int32), ("device", C.c_int32),
                ("stream", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32),
                ("synth_seed", C.c_uint64), ("attn_variant", C.c_int32), ("compact_mode", C.c_int32),
                ("compact_policy", C.c_int32), ("num_kv_heads", C.c_int32), ("reserve_sms", C.c_int32)]


class s3_buffers(C.Structure):
    _fields_ = [("arena", C.c_void_p), ("arena_bytes", C.c_int64),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64),
                ("staging", C.c_void_p), ("staging_bytes", C.c_int64),
                ("host_store", C.c_void_p), ("host_store_bytes", C.c_int64)]


class s3_request(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("prompt_len", C.c_int32), ("alloc_out", C.c_int32)]


class s3_evicted(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("batch_index", C.c_int32), ("prompt_len", C.c_int32),
                ("gen_len", C.c_int32), ("len", C.c_int32), ("cap_rows", C.c_int32),
                ("new_cap_rows", C.c_int32), ("host_off", C.c_int64)]


class s3_evict_report(C.Structure):
    _fields_ = [("n_before", C.c_int32), ("n_finished", C.c_int32), ("n_evicted", C.c_int32),
                ("n_kept", C.c_int32), ("tail_rows", C.c_int64), ("d2h_bytes", C.c_int64),
                ("moved_bytes", C.c_int64), ("paper_pcie_bytes", C.c_int64),
                ("paper_hbm_bytes", C.c_int64), ("first_hole", C.c_int32), ("sync_evict", C.c_int32)]


class s3_admit_report(C.Structure):
    _fields_ = [("n_admitted", C.c_int32), ("n_fresh", C.c_int32), ("n_reloaded", C.c_int32),
                ("n_batch", C.c_int32), ("tail_rows", C.c_int64), ("fill_bytes", C.c_int64),
                ("h2d_bytes", C.c_int64), ("moved_bytes", C.c_int64), ("stage_reload_bytes", C.c_int64)]


class s3_counters(C.Structure):
    _fields_ = [("world", C.c_int32), ("exchanges", C.c_int32),
                ("rank_free_rows", C.c_int64 * S3_MAX_RANKS), ("rank_running", C.c_int64 * S3_MAX_RANKS),
                ("free_rows_total", C.c_int64), ("running_total", C.c_int64), ("evicted_waiting_total", C.c_int64),
                ("fresh_waiting", C.c_int64), ("finished_total", C.c_int64), ("evicted_total", C.c_int64),
                ("tokens_total", C.c_int64)]


class s3_slot(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("prompt_len", C.c_int32), ("gen_len", C.c_int32),
                ("len", C.c_int32), ("cap_rows", C.c_int32), ("off", C.c_int64)]


class s3_profile(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("attn_launches", C.c_int64), ("move_launches", C.c_int64),
                ("fused_steps", C.c_int64), ("attn_ms", C.c_double), ("move_ms", C.c_double),
                ("attn_bytes", C.c_double), ("move_bytes", C.c_double), ("fused_move_bytes", C.c_double),
                ("d2h_copies", C.c_int64), ("h2d_copies", C.c_int64), ("d2h_ms", C.c_double),
                ("d2h_bytes", C.c_double), ("h2d_ms", C.c_double), ("h2d_bytes", C.c_double),
                ("d2h_overlap_ms", C.c_double), ("prep_launches", C.c_int64), ("prep_ms", C.c_double)]


class s3_gemm_args(C.Structure):
    _fields_ = [("a", C.c_void_p), ("w", C.c_void_p), ("d", C.c_void_p * 3), ("c", C.c_void_p),
                ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("seg_cols", C.c_int32), ("epi", C.c_int32),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64)]


class s3_host_io(C.Structure):
    _fields_ = [("q", C.c_void_p), ("k_new", C.c_void_p), ("v_new", C.c_void_p), ("eos", C.c_void_p),
                ("out", C.c_void_p), ("q_dev", C.c_void_p), ("k_new_dev", C.c_void_p),
                ("v_new_dev", C.c_void_p), ("eos_dev", C.c_void_p), ("chunks", C.c_int32),
                ("out_dev", C.c_void_p)]


P = C.c_void_p
_i32, _i64 = C.c_int32, C.c_int64
_SIGS = {
    "s3_workspace_query": (C.c_int, [P, P, P, P, P]),
    "s3_kv_init": (C.c_int, [P, P, P]),
    "s3_kv_destroy": (C.c_int, [P]),
    "s3_last_error": (C.c_char_p, [P]),
    "s3_submit": (C.c_int, [P, P, _i32]),
    "s3_decode_step": (C.c_int, [P, _i32, _i32, P, P, P, P, P]),
    "s3_decode_step_host": (C.c_int, [P, P]),
    "s3_evict_compact": (C.c_int, [P, P, P, P, P]),
    "s3_evict_wait": (C.c_int, [P]),
    "s3_admit": (C.c_int, [P, P, P]),
    "s3_admit_home": (C.c_int, [P, P, P]),
    "s3_admit_shared": (C.c_int, [P, P, P, P]),
    "s3_counters_local": (C.c_int, [P, P]),
    "s3_evict_wait_req": (C.c_int, [P, _i64]),
    "s3_nccl_get_unique_id": (C.c_int, [P]),
    "s3_comm_init": (C.c_int, [P, P]),
    "s3_exchange_counters": (C.c_int, [P, P]),
    "s3_counters_get": (C.c_int, [P, P]),
    "s3_plan_ffd": (_i32, [_i32, P, P, _i64, _i32, P]),
    "s3_plan_ffd_multibin": (_i32, [_i32, P, P, _i32, P, P, P]),
    "s3_batch_size": (C.c_int, [P, P]),
    "s3_batch_view": (C.c_int, [P, P, P]),
    "s3_profile_enable": (C.c_int, [P, _i32]),
    "s3_profile_get": (C.c_int, [P, P]),
    "s3_synth_inputs": (C.c_int, [P, _i32, _i32, P, _i64, P, P, P, P]),
    "s3_verify_resident": (C.c_int, [P, P]),
    "s3_gemm": (C.c_int, [P, P]),
    "s3_gemm_workspace": (C.c_int, [P, P]),
    "s3_cast_bf16": (C.c_int, [P, P, P, _i64]),
}

_lib = None


def header_functions() -> list[str]:
    """Function names declared in include/s3.h (for the export check)."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(s3_[a-z_0-9]+)\s*\(", txt)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libs3.so not built ({LIB_PATH}); run __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    return C.cast(x, C.c_void_p).value


def _check(rc: int, where: str, ctx=None):
    if rc != S3_OK:
        msg = lib().s3_last_error(ctx).decode() if ctx else ""
        raise S3Error(rc, where, msg)


# ---- same-named wrappers ----------------------------------------------------

def s3_workspace_query(cfg: s3_config):
    a, w, s, h = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().s3_workspace_query(C.byref(cfg), C.byref(a), C.byref(w), C.byref(s), C.byref(h)),
           "s3_workspace_query")
    return a.value, w.value, s.value, h.value


def s3_kv_init(cfg: s3_config, bufs: s3_buffers):
    ctx = C.c_void_p()
    _check(lib().s3_kv_init(C.byref(cfg), C.byref(bufs), C.byref(ctx)), "s3_kv_init")
    return ctx


def s3_kv_destroy(ctx):
    _check(lib().s3_kv_destroy(ctx), "s3_kv_destroy")


def s3_submit(ctx, reqs):
    """reqs: ctypes array of s3_request."""
    _check(lib().s3_submit(ctx, C.cast(reqs, C.c_void_p), len(reqs)), "s3_submit", ctx)


def s3_decode_step(ctx, l0, nl, q, k_new, v_new, eos, out):
    _check(lib().s3_decode_step(ctx, l0, nl, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(eos), _ptr(out)),
           "s3_decode_step", ctx)


def s3_decode_step_host(ctx, q, k_new, v_new, eos, out, q_dev, k_new_dev, v_new_dev, eos_dev, chunks=0,
                        out_dev=None):
    """q/k_new/v_new/eos/out: pinned host tensors; *_dev: device landing buffers
    (out_dev None: the kernels store `out` over PCIe)."""
    io = s3_host_io(_ptr(q), _ptr(k_new), _ptr(v_new), _ptr(eos), _ptr(out), _ptr(q_dev), _ptr(k_new_dev),
                    _ptr(v_new_dev), _ptr(eos_dev), int(chunks), _ptr(out_dev))
    _check(lib().s3_decode_step_host(ctx, C.byref(io)), "s3_decode_step_host", ctx)


def s3_evict_compact(ctx, n_before: int):
    rep = s3_evict_report()
    n = max(n_before, 1)
    perm = (C.c_int32 * n)()
    ev = (s3_evicted * n)()
    fin = (C.c_int64 * n)()
    _check(lib().s3_evict_compact(ctx, C.byref(rep), C.cast(perm, P), C.cast(ev, P), C.cast(fin, P)),
           "s3_evict_compact", ctx)
    return rep, list(perm[:rep.n_before]), list(ev[:rep.n_evicted]), list(fin[:rep.n_finished])


def s3_evict_wait(ctx):
    _check(lib().s3_evict_wait(ctx), "s3_evict_wait", ctx)


def s3_evict_wait_req(ctx, req_id: int):
    _check(lib().s3_evict_wait_req(ctx, int(req_id)), "s3_evict_wait_req", ctx)


def _admit(fn, name, ctx, cap, *args):
    rep = s3_admit_report()
    ids = (C.c_int64 * max(cap, 1))()
    _check(fn(ctx, *args, C.byref(rep), C.cast(ids, P)), name, ctx)
    return rep, list(ids[:rep.n_admitted])


def s3_admit(ctx, max_running: int):
    return _admit(lib().s3_admit, "s3_admit", ctx, max_running)


def s3_admit_home(ctx, max_running: int):
    return _admit(lib().s3_admit_home, "s3_admit_home", ctx, max_running)


def s3_admit_shared(ctx, max_running: int, counters_all):
    """counters_all: int64 numpy array [world, S3_NCOUNTERS] (contiguous)."""
    return _admit(lib().s3_admit_shared, "s3_admit_shared", ctx, max_running, _ptr(counters_all))


def s3_counters_local(ctx, row):
    """row: int64 numpy array [S3_NCOUNTERS]."""
    _check(lib().s3_counters_local(ctx, _ptr(row)), "s3_counters_local", ctx)


def s3_nccl_get_unique_id() -> bytes:
    buf = (C.c_uint8 * S3_NCCL_ID_BYTES)()
    _check(lib().s3_nccl_get_unique_id(C.cast(buf, P)), "s3_nccl_get_unique_id", None)
    return bytes(buf)


def s3_comm_init(ctx, uid: bytes):
    assert len(uid) == S3_NCCL_ID_BYTES
    buf = (C.c_uint8 * S3_NCCL_ID_BYTES).from_buffer_copy(uid)
    _check(lib().s3_comm_init(ctx, C.cast(buf, P)), "s3_comm_init", ctx)


def s3_exchange_counters(ctx, counters_all):
    """counters_all: int64 numpy array [world, S3_NCOUNTERS] (contiguous), overwritten."""
    _check(lib().s3_exchange_counters(ctx, _ptr(counters_all)), "s3_exchange_counters", ctx)


def s3_counters_get(ctx) -> s3_counters:
    c = s3_counters()
    _check(lib().s3_counters_get(ctx, C.byref(c)), "s3_counters_get", ctx)
    return c


def s3_plan_ffd(cap, req, free_rows, max_items, admitted):
    return lib().s3_plan_ffd(len(cap), _ptr(cap), _ptr(req), int(free_rows), int(max_items), _ptr(admitted))


def s3_plan_ffd_multibin(cap, req, free_rows, free_slots, rank):
    return lib().s3_plan_ffd_multibin(len(cap), _ptr(cap), _ptr(req), len(free_rows), _ptr(free_rows),
                                      _ptr(free_slots), _ptr(rank))


def s3_batch_size(ctx) -> int:
    b = C.c_int32()
    _check(lib().s3_batch_size(ctx, C.byref(b)), "s3_batch_size", ctx)
    return b.value


def s3_batch_view(ctx):
    B = s3_batch_size(ctx)
    arr = (s3_slot * max(B, 1))()
    b = C.c_int32()
    _check(lib().s3_batch_view(ctx, C.cast(arr, P), C.byref(b)), "s3_batch_view", ctx)
    return [(s.req_id, s.prompt_len, s.gen_len, s.len, s.cap_rows, s.off) for s in arr[:b.value]]


def s3_profile_enable(ctx, on: bool):
    _check(lib().s3_profile_enable(ctx, 1 if on else 0), "s3_profile_enable", ctx)


def s3_profile_get(ctx) -> s3_profile:
    p = s3_profile()
    _check(lib().s3_profile_get(ctx, C.byref(p)), "s3_profile_get", ctx)
    return p


def s3_synth_inputs(ctx, l0, nl, out_len_by_req, q, k_new, v_new, eos):
    _check(lib().s3_synth_inputs(ctx, l0, nl, _ptr(out_len_by_req), int(out_len_by_req.numel()),
                                 _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(eos)), "s3_synth_inputs", ctx)


def s3_verify_resident(ctx) -> int:
    bad = C.c_int64()
    _check(lib().s3_verify_resident(ctx, C.byref(bad)), "s3_verify_resident", ctx)
    return bad.value


def s3_gemm(stream, a, w, d, c=None, epi=0, seg_cols=None, workspace=None, M=None):
    """D = epi(A . W^T) on the tensor cores (include/s3.h s3_gemm).  a: [M][K]
    bf16, w: [N][K] bf16, d: one [M][N] tensor or a list of up to 3 column
    segments [M][seg_cols]; epi 0 store, 1 gelu_tanh, 2 add c; workspace: a
    zero-initialised uint8 device tensor for split-K (or None)."""
    segs = list(d) if isinstance(d, (list, tuple)) else [d]
    M = int(a.shape[-2] if M is None else M)
    K = a.shape[-1]
    N = w.shape[0]
    g = s3_gemm_args()
    if workspace is not None:
        g.workspace, g.workspace_bytes = _ptr(workspace), int(workspace.numel())
    g.a, g.w = _ptr(a), _ptr(w)
    for i, t in enumerate(segs):
        g.d[i] = _ptr(t)
    g.c = _ptr(c)
    g.M, g.N, g.K, g.epi = int(M), int(N), int(K), int(epi)
    g.seg_cols = int(seg_cols if seg_cols is not None else N // len(segs))
    _check(lib().s3_gemm(_ptr(stream) if not hasattr(stream, "cuda_stream") else stream.cuda_stream,
                         C.byref(g)), "s3_gemm")


def s3_cast_bf16(stream, src, dst, n=None):
    """dst (bf16) = src (fp32), n elements (default: src.numel())."""
    n = int(src.numel() if n is None else n)
    _check(lib().s3_cast_bf16(stream.cuda_stream if hasattr(stream, "cuda_stream") else _ptr(stream), _ptr(src),
                              _ptr(dst), n), "s3_cast_bf16")


def s3_gemm_workspace(M, N, K, seg_cols=None, epi=0) -> int:
    g = s3_gemm_args()
    g.M, g.N, g.K, g.epi = int(M), int(N), int(K), int(epi)
    g.seg_cols = int(seg_cols or N)
    out = C.c_int64()
    _check(lib().s3_gemm_workspace(C.byref(g), C.byref(out)), "s3_gemm_workspace")
    return int(out.value)

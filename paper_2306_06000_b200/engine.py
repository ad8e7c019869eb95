"""S3Engine: buffer allocation (torch) + the per-iteration call sequence.

This is the public Python API a user drives.  It allocates the caller-owned
buffers of include/s3.h with torch (device memory, pinned host memory, the
current stream) and calls the four ABI entry points in the order the paper's
iteration-level loop implies:

    decode (attention + append + detect) -> evict + compact -> admit

Every step of the method runs inside libs3.so; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import s3 as abi


@dataclass
class StepStats:
    batch: int
    tokens: int
    finished: int
    evicted: int
    admitted: int
    d2h_bytes: int
    moved_bytes: int
    paper_pcie_bytes: int
    paper_hbm_bytes: int
    reload_bytes: int
    fill_bytes: int
    stage_reload_bytes: int = 0


class S3Engine:
    def __init__(self, num_layers, num_heads, head_dim, max_seq_len, arena_rows, max_running,
                 chunk_rows=0, move_chunk_bytes=0, device=0, rank=0, world=1, seed=1,
                 staging_bytes=None, host_store_bytes=None, io_rows=None, attn_variant=0, compact_mode=0,
                 compact_policy=0, num_kv_heads=0, reserve_sms=0, exchange_admission=False):
        if not torch.cuda.is_available():
            raise RuntimeError("S3Engine needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.L, self.H, self.D = num_layers, num_heads, head_dim
        self.Hkv = num_kv_heads or num_heads
        self.max_running = max_running
        self.world, self.rank = world, rank
        # the multi-rank admission (home re-admission -> counter all-reduce -> shared multi-bin
        # FFD) also at world 1 when asked: with one bin it admits exactly what s3_admit does,
        # and it puts the caller's process-group exchange (NCCL) on the step's path
        self.split_admit = world > 1 or exchange_admission
        self.native_comm = False        # counters all-reduced by libs3's own NCCL communicator
        self.stream = torch.cuda.current_stream(self.device)
        self.cfg = abi.s3_config(
            num_layers=num_layers, num_heads=num_heads, head_dim=head_dim, max_seq_len=max_seq_len,
            arena_rows=arena_rows, max_running=max_running, chunk_rows=chunk_rows,
            move_chunk_bytes=move_chunk_bytes, device=device, stream=self.stream.cuda_stream,
            rank=rank, world=world, synth_seed=seed, attn_variant=attn_variant, compact_mode=compact_mode,
            compact_policy=compact_policy, num_kv_heads=num_kv_heads, reserve_sms=reserve_sms)
        arena_b, ws_b, st_min, hs_min = abi.s3_workspace_query(self.cfg)
        self.kvpt = 4 * num_layers * self.Hkv * head_dim
        self.arena = torch.empty(arena_b, dtype=torch.uint8, device=self.device)
        self.workspace = torch.empty(ws_b, dtype=torch.uint8, device=self.device)
        st_b = st_min if staging_bytes is None else staging_bytes
        self.staging = torch.empty(max(st_b, 16), dtype=torch.uint8, device=self.device)
        hs_b = max(hs_min, host_store_bytes or 4 * hs_min)
        self.host_store = torch.empty(hs_b, dtype=torch.uint8, pin_memory=True)
        bufs = abi.s3_buffers(self.arena.data_ptr(), arena_b, self.workspace.data_ptr(), ws_b,
                              self.staging.data_ptr() if st_b > 0 else None, st_b,
                              self.host_store.data_ptr(), hs_b)
        self.ctx = abi.s3_kv_init(self.cfg, bufs)
        rows = io_rows or max_running
        n = num_layers * rows * num_heads * head_dim
        nk = num_layers * rows * self.Hkv * head_dim
        self.q = torch.empty(n, dtype=torch.bfloat16, device=self.device)
        self.k_new = torch.empty(nk, dtype=torch.bfloat16, device=self.device)
        self.v_new = torch.empty(nk, dtype=torch.bfloat16, device=self.device)
        self.out = torch.empty(n, dtype=torch.float32, device=self.device)
        self.eos = torch.empty(max(rows, 1), dtype=torch.uint8, device=self.device)
        self.out_len = None
        self._out_len_h = None
        self.max_seq_len = max_seq_len
        self.counters = np.zeros(abi.S3_NCOUNTERS, np.int64)

    # ---- lifecycle -----------------------------------------------------
    def close(self):
        """Destroy the context and drop every caller-owned buffer (the device
        memory returns to torch's allocator once no other reference holds it)."""
        if getattr(self, "ctx", None):
            abi.s3_kv_destroy(self.ctx)
            self.ctx = None
        for name in ("arena", "workspace", "staging", "host_store", "q", "k_new", "v_new", "out", "eos", "out_len"):
            if hasattr(self, name):
                setattr(self, name, None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- pool ----------------------------------------------------------
    def submit(self, req_id, prompt, alloc, out_len=None):
        """Submit requests; out_len (actual output lengths) feeds only the
        synthetic sampler stand-in (s3_synth_inputs), never the method."""
        n = len(req_id)
        arr = (abi.s3_request * n)()
        for i in range(n):
            arr[i].req_id = int(req_id[i])
            arr[i].prompt_len = int(prompt[i])
            arr[i].alloc_out = int(alloc[i])
        abi.s3_submit(self.ctx, arr)
        # the sampler stand-in's table (indexed by req_id), kept across submit calls;
        # requests without an out_len run to the maximum length (R28)
        ids = np.asarray(req_id, np.int64)
        if n == 0:
            return
        need = int(ids.max()) + 1
        if self._out_len_h is None or self._out_len_h.shape[0] < need:
            grown = np.zeros(max(need, 2 * (0 if self._out_len_h is None else self._out_len_h.shape[0])), np.int32)
            if self._out_len_h is not None:
                grown[:self._out_len_h.shape[0]] = self._out_len_h
            self._out_len_h = grown
        self._out_len_h[ids] = (np.asarray(out_len, np.int32) if out_len is not None
                                else self.max_seq_len - np.asarray(prompt, np.int32))
        self.out_len = torch.from_numpy(self._out_len_h).to(self.device)

    # ---- the four calls --------------------------------------------------
    @property
    def B(self) -> int:
        return abi.s3_batch_size(self.ctx)

    def synth_inputs(self, l0=0, nl=None):
        nl = self.L - l0 if nl is None else nl
        abi.s3_synth_inputs(self.ctx, l0, nl, self.out_len, self.q, self.k_new, self.v_new, self.eos)

    def decode(self, l0=0, nl=None, q=None, k_new=None, v_new=None, eos=None, out=None):
        nl = self.L - l0 if nl is None else nl
        abi.s3_decode_step(self.ctx, l0, nl, self.q if q is None else q, self.k_new if k_new is None else k_new,
                           self.v_new if v_new is None else v_new, self.eos if eos is None else eos,
                           self.out if out is None else out)

    def decode_host(self, q, k_new, v_new, eos, out, chunks=0, device_out=True):
        """Whole decode step fed from pinned HOST tensors (s3_decode_step_host):
        q/k_new/v_new/eos are copied into this engine's device buffers inside
        the call, pipelined with the attention kernel; `out` (pinned fp32) is
        filled by per-chunk D2H copies from this engine's device `out`
        (device_out) or stored by the kernels directly over PCIe.
        Synchronise the stream before reading `out`."""
        abi.s3_decode_step_host(self.ctx, q, k_new, v_new, eos, out, self.q, self.k_new, self.v_new, self.eos,
                                chunks, self.out if device_out else None)

    def evict_compact(self):
        return abi.s3_evict_compact(self.ctx, self.B)

    def admit(self):
        if self.world == 1:
            return abi.s3_admit(self.ctx, self.max_running)
        raise RuntimeError("world > 1: use admit_home / exchange / admit_shared")

    # ---- (a8) the counter exchange over libs3's NCCL communicator ------------------
    def comm_init(self, uid: bytes):
        """Bind the library-owned NCCL communicator (collective over the ranks; uid from
        abi.s3_nccl_get_unique_id on rank 0, broadcast by the caller)."""
        abi.s3_comm_init(self.ctx, uid)
        self.native_comm = True

    def exchange_counters(self) -> np.ndarray:
        mat = np.zeros((self.world, abi.S3_NCOUNTERS), np.int64)
        abi.s3_exchange_counters(self.ctx, mat)
        return mat

    def counters_get(self):
        return abi.s3_counters_get(self.ctx)

    def _exchange(self, exchange):
        if exchange is None:           # libs3's communicator (comm_init) does the all-reduce
            if not self.native_comm:
                raise RuntimeError("world > 1: pass an exchange callable or call comm_init first")
            return self.exchange_counters()
        return exchange(self.counters_local())

    def admit_step(self, exchange=None):
        """The step's admission: s3_admit (world 1), or s3_admit_home, the all-reduce of the
        counter rows (the caller's `exchange`, or with none libs3's communicator after
        comm_init), s3_admit_shared.  Returns the admission reports."""
        if not self.split_admit:
            return [self.admit()[0]]
        hrep, _ = self.admit_home()
        srep, _ = self.admit_shared(self._exchange(exchange))
        return [hrep, srep]

    def admit_home(self):
        return abi.s3_admit_home(self.ctx, self.max_running)

    def counters_local(self) -> np.ndarray:
        abi.s3_counters_local(self.ctx, self.counters)
        return self.counters.copy()

    def admit_shared(self, counters_all: np.ndarray):
        return abi.s3_admit_shared(self.ctx, self.max_running, np.ascontiguousarray(counters_all, np.int64))

    def batch_view(self):
        return abi.s3_batch_view(self.ctx)

    def verify_resident(self) -> int:
        return abi.s3_verify_resident(self.ctx)

    def evict_wait(self):
        abi.s3_evict_wait(self.ctx)

    def evict_wait_req(self, req_id: int):
        abi.s3_evict_wait_req(self.ctx, req_id)

    def profile(self, on: bool):
        abi.s3_profile_enable(self.ctx, on)

    def profile_get(self):
        return abi.s3_profile_get(self.ctx)

    # ---- one iteration (world == 1) ---------------------------------------
    def step(self, exchange=None) -> StepStats:
        """synth inputs -> decode -> evict+compact -> admit.  `exchange` is a
        callable(local_row int64[8]) -> all rows int64[world, 8] (an
        all-reduce done by the caller's process group) used when world > 1."""
        B = self.B
        if B:
            self.synth_inputs()
        self.decode()
        rep, perm, ev, fin = self.evict_compact()
        reps = self.admit_step(exchange)
        return StepStats(B, B, rep.n_finished, rep.n_evicted, sum(r.n_admitted for r in reps), rep.d2h_bytes,
                         rep.moved_bytes + sum(r.moved_bytes for r in reps), rep.paper_pcie_bytes,
                         rep.paper_hbm_bytes, sum(r.h2d_bytes for r in reps), sum(r.fill_bytes for r in reps),
                         sum(r.stage_reload_bytes for r in reps))

    def initial_admit(self, exchange=None):
        if not self.split_admit:
            return self.admit()
        self.admit_home()
        return self.admit_shared(self._exchange(exchange))

    def arena_rows_view(self) -> torch.Tensor:
        """The arena as bf16 [R][L][2][H][D] (a view, no copy)."""
        R = self.cfg.arena_rows                    # (the allocation ends with 8 guard rows)
        return self.arena[:R * self.kvpt].view(torch.bfloat16).view(R, self.L, 2, self.Hkv, self.D)

    def host_rows(self, host_off: int, rows: int) -> torch.Tensor:
        n = rows * self.kvpt
        return self.host_store[host_off:host_off + n].view(torch.bfloat16).view(rows, self.L, 2, self.Hkv, self.D)

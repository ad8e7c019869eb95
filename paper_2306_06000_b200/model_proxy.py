"""GPT-J-shaped random-weight decoder around the S^3 hot path.

The paper's throughput gap between ORCA (max-length reservation), S^3 and
the Oracle comes from batching: the feed-forward and projection GEMMs share
their weights across the batch while self-attention does not
(PAPER.md:247-249, 168).  This proxy puts that batch-dependent cost around
the decode step: per layer, QKV projection -> s3_decode_step(l, 1) ->
output projection + feed-forward (GPT-J's parallel residual), with random
bf16 weights of GPT-J-6B's shapes (d = 4096, 16 heads x 256, FFN 16384,
28 layers; ~11.3 GB).  The GEMMs are plain library GEMMs (cuBLAS through
torch.matmul); the attention, append, detection, eviction, compaction and
admission stay in libs3.so.  No trained weights are involved: outputs are
not text, only the timing is meaningful.
"""
from __future__ import annotations

import math

import torch

from .engine import S3Engine


class GPTJProxy:
    def __init__(self, eng: S3Engine, d_ff: int = 16384, seed: int = 0):
        self.eng = eng
        L, H, D = eng.L, eng.H, eng.D
        self.d = H * D
        self.d_ff = d_ff
        dev = eng.device
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        s_in = 1.0 / math.sqrt(self.d)
        s_ff = 1.0 / math.sqrt(d_ff)

        def w(rows, cols, scale):
            return (torch.randn(rows, cols, device=dev, dtype=torch.bfloat16, generator=g) * scale)

        self.w_qkv = [w(self.d, 3 * self.d, s_in) for _ in range(L)]
        self.w_o = [w(self.d, self.d, s_in) for _ in range(L)]
        self.w_1 = [w(self.d, d_ff, s_in) for _ in range(L)]
        self.w_2 = [w(d_ff, self.d, s_ff) for _ in range(L)]
        self.x0 = torch.randn(eng.max_running, self.d, device=dev, dtype=torch.bfloat16, generator=g)
        self.qkv = torch.empty(eng.max_running, 3 * self.d, device=dev, dtype=torch.bfloat16)

    @property
    def weight_bytes(self) -> int:
        per = 3 * self.d * self.d + self.d * self.d + 2 * self.d * self.d_ff
        return 2 * per * self.eng.L

    def flops(self, B: int) -> float:
        """GEMM flops of one decode step at batch B (attention excluded)."""
        per = 3 * self.d * self.d + self.d * self.d + 2 * self.d * self.d_ff
        return 2.0 * B * per * self.eng.L

    def decode_step(self):
        """One token for every running slot: 28 x (QKV GEMM -> attention ->
        O + FFN GEMMs).  eos comes from the synthetic sampler stand-in."""
        eng = self.eng
        B = eng.B
        L, H, D = eng.L, eng.H, eng.D
        HD = H * D
        if B:
            # sampler stand-in: eos (and the last layer's synthetic q/k/v, overwritten below)
            eng.synth_inputs(L - 1, 1)
            x = self.x0[:B].clone()
        for l in range(L):
            if B:
                qkv = self.qkv[:B]
                torch.matmul(x, self.w_qkv[l], out=qkv)
                q = eng.q[:B * HD].view(B, HD)
                k = eng.k_new[:B * HD].view(B, HD)
                v = eng.v_new[:B * HD].view(B, HD)
                q.copy_(qkv[:, :HD])
                k.copy_(qkv[:, HD:2 * HD])
                v.copy_(qkv[:, 2 * HD:])
            eng.decode(l, 1, q=eng.q, k_new=eng.k_new, v_new=eng.v_new, eos=eng.eos, out=eng.out)
            if B:
                a = eng.out[:B * HD].view(B, HD).to(torch.bfloat16)
                hdn = torch.nn.functional.gelu(x @ self.w_1[l], approximate="tanh")
                x = x + a @ self.w_o[l] + hdn @ self.w_2[l]
        return B

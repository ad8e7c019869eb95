"""GPT-J-shaped random-weight decoder around the S^3 hot path.

The paper's throughput gap between ORCA (max-length reservation), S^3 and
the Oracle comes from batching: the feed-forward and projection GEMMs share
their weights across the batch while self-attention does not
(PAPER.md:247-249, 168).  This proxy puts that batch-dependent cost around
the decode step: per layer, QKV projection -> s3_decode_step(l, 1) ->
output projection + feed-forward (GPT-J's parallel residual), with random
bf16 weights of GPT-J-6B's shapes (d = 4096, 16 heads x 256, FFN 16384,
28 layers; ~11.3 GB).

Every GEMM is libs3's tcgen05 kernel (s3_gemm): the QKV projection writes
q, k_new and v_new straight into the engine's decode buffers (three column
segments), the FFN up-projection applies GELU in its epilogue and the output
and down projections add into the residual stream in theirs; the attention
output is cast to bf16 by s3_cast_bf16.  torch only allocates.  LayerNorm and
rotary embeddings are omitted (R24): no trained weights are
involved, outputs are not text, only the timing (and the kernels' numerics,
tests/test_gpu_gemm.py) are meaningful.
"""
from __future__ import annotations

import math

import torch

from . import s3 as abi
from .engine import S3Engine


class GPTJProxy:
    def __init__(self, eng: S3Engine, d_ff: int = 16384, seed: int = 0):
        self.eng = eng
        L, H, D = eng.L, eng.H, eng.D
        if eng.Hkv != H:
            raise ValueError("the GPT-J proxy has multi-head KV (num_kv_heads = num_heads)")
        self.d = H * D
        self.d_ff = d_ff
        dev = eng.device
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        s_in = 1.0 / math.sqrt(self.d)
        s_ff = 1.0 / math.sqrt(d_ff)

        def w(out_f, in_f, scale):           # nn.Linear layout [out][in] (K-major for s3_gemm)
            return (torch.randn(out_f, in_f, device=dev, dtype=torch.bfloat16, generator=g) * scale)

        self.w_qkv = [w(3 * self.d, self.d, s_in) for _ in range(L)]
        self.w_o = [w(self.d, self.d, s_in) for _ in range(L)]
        self.w_1 = [w(d_ff, self.d, s_in) for _ in range(L)]
        self.w_2 = [w(self.d, d_ff, s_ff) for _ in range(L)]
        self.x0 = torch.randn(eng.max_running, self.d, device=dev, dtype=torch.bfloat16, generator=g)
        self.x = torch.empty(eng.max_running, self.d, device=dev, dtype=torch.bfloat16)
        self.a = torch.empty(eng.max_running, self.d, device=dev, dtype=torch.bfloat16)
        self.h = torch.empty(eng.max_running, d_ff, device=dev, dtype=torch.bfloat16)
        # split-K scratch of s3_gemm (small batches spread K over idle SMs); zeroed once
        self.ws = torch.zeros(96 << 20, device=dev, dtype=torch.uint8)

    @property
    def weight_bytes(self) -> int:
        per = 3 * self.d * self.d + self.d * self.d + 2 * self.d * self.d_ff
        return 2 * per * self.eng.L

    def flops(self, B: float) -> float:
        """GEMM flops of one decode step at batch B (attention excluded)."""
        per = 3 * self.d * self.d + self.d * self.d + 2 * self.d * self.d_ff
        return 2.0 * B * per * self.eng.L

    def layer_gemms(self, l: int, B: int, stream):
        """The four projections of layer l around its attention (x: [B][d])."""
        eng, HD, ws = self.eng, self.d, self.ws
        x, a, h = self.x[:B], self.a[:B], self.h[:B]
        return (
            # QKV straight into the decode buffers: [nl = 1][B][H][D] each
            lambda: abi.s3_gemm(stream, x, self.w_qkv[l],
                                [eng.q[:B * HD], eng.k_new[:B * HD], eng.v_new[:B * HD]], seg_cols=HD, workspace=ws),
            # attention out (fp32) -> bf16, then x += a Wo^T ; h = gelu(x Wi^T) ; x += h W2^T
            lambda: (abi.s3_cast_bf16(stream, eng.out, a, B * HD),
                     abi.s3_gemm(stream, x, self.w_1[l], h, epi=1, workspace=ws),
                     abi.s3_gemm(stream, a, self.w_o[l], x, c=x, epi=2, workspace=ws),
                     abi.s3_gemm(stream, h, self.w_2[l], x, c=x, epi=2, workspace=ws)),
        )

    def decode_step(self, on_layer=None):
        """One token for every running slot: L x (QKV GEMM -> attention ->
        O + FFN GEMMs).  eos comes from the synthetic sampler stand-in.
        on_layer(l, B) (tests) runs after each layer's attention."""
        eng = self.eng
        B = eng.B
        L = eng.L
        stream = eng.stream
        if B:
            # sampler stand-in: eos (and the last layer's synthetic q/k/v, overwritten below)
            eng.synth_inputs(L - 1, 1)
            self.x[:B].copy_(self.x0[:B])
        for l in range(L):
            pre, post = self.layer_gemms(l, B, stream) if B else (None, None)
            if B:
                pre()
            eng.decode(l, 1, q=eng.q, k_new=eng.k_new, v_new=eng.v_new, eos=eng.eos, out=eng.out)
            if on_layer is not None:
                on_layer(l, B)
            if B:
                # GPT-J parallel residual: both branches read the layer's input x; the
                # FFN up-projection runs before x is updated in place
                post()
        return B

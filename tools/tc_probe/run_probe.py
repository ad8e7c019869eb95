"""Build and run the tcgen05 probe; compare with torch (fp32)."""
import ctypes as C
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libtcprobe.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                       "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(HERE, "tc_probe.cu")])
lib = C.CDLL(LIB)
torch.manual_seed(0)
dev = torch.device("cuda")
pitch = 512                                  # K rows with a wider pitch (like a KV head inside a row)
Kbig = torch.randn(128, pitch // 2, device=dev).to(torch.bfloat16)
K = Kbig[:, :128]
Q = torch.randn(16, 128, device=dev).to(torch.bfloat16)
V = torch.randn(128, 128, device=dev).to(torch.bfloat16)
P = torch.rand(16, 128, device=dev)
s_out = torch.zeros(128, 16, device=dev)
o_out = torch.zeros(128, 16, device=dev)
rc = lib.tc_probe_run(C.c_void_p(Kbig.data_ptr()), C.c_void_p(Q.data_ptr()), C.c_void_p(V.data_ptr()),
                      C.c_void_p(P.data_ptr()), C.c_void_p(s_out.data_ptr()), C.c_void_p(o_out.data_ptr()),
                      C.c_int(pitch))
print("rc", rc)
S_ref = K.float() @ Q.float().t()
O_ref = V.float().t() @ P.to(torch.bfloat16).float().t()
print("S max err", (s_out - S_ref).abs().max().item(), "ref max", S_ref.abs().max().item())
print("O max err", (o_out - O_ref).abs().max().item(), "ref max", O_ref.abs().max().item())
print("S sample", s_out[0, :4].tolist(), S_ref[0, :4].tolist())
print("O sample", o_out[0, :4].tolist(), O_ref[0, :4].tolist())
ok = (s_out - S_ref).abs().max().item() < 1e-2 and (o_out - O_ref).abs().max().item() < 1e-2
print("PROBE", "OK" if ok else "FAIL")

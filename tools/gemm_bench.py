"""Grouped DMMA GEMM vs cuBLAS DGEMM on the same shapes (run under ncu for the
kernel durations of the library's GEMM; torch events time cuBLAS)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_11932_b200 as tg  # noqa: E402

shapes = [(1024, 1024, 2048, 0, 1), (1024, 1024, 512, 0, 1), (512, 512, 350, 0, 1),
          (4096, 4096, 4096, 0, 0), (8192, 32, 512, 0, 0), (512, 32, 512, 1, 0)]
for M, N, K, ta, tb in shapes:
    r = np.random.default_rng(0)
    A = r.normal(size=(K, M) if ta else (M, K))
    B = r.normal(size=(N, K) if tb else (K, N))
    for _ in range(3):
        tg.tlr.gemm(1.0, A, ta, B, tb)
    At = torch.tensor(A, device="cuda")
    Bt = torch.tensor(B, device="cuda")
    a = At.T if ta else At
    b = Bt.T if tb else Bt
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{M}x{N}x{K} ta={ta} tb={tb}: cuBLAS {ms*1e3:.1f} us = {2*M*N*K/ms/1e9:.2f} TF/s", flush=True)

"""Input-layer dense ops of the papers100M-shaped step, timed alone (CUDA
events, warm, TF32 as in the engine) against their HBM floor, with the
alternative formulations cuBLAS offers.

    python scripts/gemm_probe.py [--rows 90112]
"""

from __future__ import annotations

import argparse
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=90112)
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = True
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    R, K, N = args.rows, 256, 256
    cat = torch.randn(R, K, device="cuda")
    W = torch.randn(K, N, device="cuda")
    b = torch.randn(N, device="cuda")
    z = torch.empty(R, N, device="cuda")
    dz = torch.randn(R, N, device="cuda")
    gW = torch.empty(K, N, device="cuda")
    C = 2048
    part = torch.empty(R // C, K, N, device="cuda")

    def floor(nbytes):
        return nbytes / peak / 1e3

    fwd_bytes = 4 * (R * K + R * N + K * N)
    wg_bytes = 4 * (R * K + R * N + K * N)
    rows = [
        ("fwd addmm(b, cat, W, out=z)", lambda: torch.addmm(b, cat, W, out=z), fwd_bytes),
        ("fwd mm(cat, W, out=z)", lambda: torch.mm(cat, W, out=z), fwd_bytes),
        ("fwd (W^T cat^T)^T", lambda: torch.mm(W.t(), cat.t(), out=z.t()), fwd_bytes),
        ("wgrad mm(cat^T, dz)", lambda: torch.mm(cat.t(), dz, out=gW), wg_bytes),
        ("wgrad bmm 2048-row chunks", lambda: torch.bmm(cat.view(-1, C, K).transpose(1, 2), dz.view(-1, C, N),
                                                        out=part), wg_bytes + 4 * part.numel()),
        ("wgrad bmm 4096-row chunks", lambda: torch.bmm(cat.view(-1, 2 * C, K).transpose(1, 2),
                                                        dz.view(-1, 2 * C, N), out=part[:R // (2 * C)]),
         wg_bytes + 2 * part.numel()),
        ("copy cat -> z (same bytes)", lambda: z.copy_(cat), 4 * 2 * R * K),
    ]
    for name, fn, nbytes in rows:
        us = timeit(fn)
        print(f"{name:34s} {us:7.1f} us   floor {floor(nbytes):6.1f} us   {nbytes / us / 1e3:7.0f} GB/s "
              f"({nbytes / us / 1e3 / peak:.2f} of peak)")


if __name__ == "__main__":
    main()

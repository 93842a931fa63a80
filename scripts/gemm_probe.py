"""Time the GraphSAGE GEMM shapes/layouts on the B200 (cuBLAS kernel choice)."""
import torch

torch.backends.cuda.matmul.allow_tf32 = True
n, k, m = 148_000, 256, 256
cat = torch.randn(n, k, device="cuda")
dz = torch.randn(n, m, device="cuda")
W = torch.randn(k, m, device="cuda")
b = torch.randn(m, device="cuda")
out = torch.empty(k, m, device="cuda")
outT = torch.empty(m, k, device="cuda")


def t(fn, reps=50):
    for _ in range(5):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e3


flop = 2 * n * k * m
for name, fn in [("fwd addmm", lambda: torch.addmm(b, cat, W)),
                 ("dW mm(cat.t, dz)", lambda: torch.mm(cat.t(), dz, out=out)),
                 ("dW^T mm(dz.t, cat)", lambda: torch.mm(dz.t(), cat, out=outT)),
                 ("dcat mm(dz, W.t)", lambda: torch.mm(dz, W.t())),
                 ("dW bf16", lambda: torch.mm(cat.t().bfloat16(), dz.bfloat16())),
                 ("dW bmm74 split-K", lambda: torch.bmm(cat.view(74, -1, k)[:, :2000].transpose(1, 2),
                                                         dz.view(74, -1, m)[:, :2000]).sum(0)),
                 ("dW bmm148 split-K", lambda: torch.bmm(cat[:148000].view(148, -1, k).transpose(1, 2),
                                                          dz[:148000].view(148, -1, m)).sum(0)),
                 ]:
    us = t(fn)
    print(f"{name:24s} {us:8.1f} us  {flop / us / 1e6:8.1f} TFLOP/s")

"""SWITCH conditional graph node around a torch GEMM (scripts for the
engine's size-switched dense ops): body k = addmm over the first k*chunk
rows, the device row count picks the body at replay.

    python scripts/switch_probe.py
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2106_06150_b200 import _lib
    torch.backends.cuda.matmul.allow_tf32 = True
    R, C, K = 176000, 8192, 23
    A = torch.randn(R, 256, device="cuda")
    W = torch.randn(256, 256, device="cuda")
    b = torch.randn(256, device="cuda")
    out = torch.zeros(R, 256, device="cuda")
    n_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
    main_s, aux = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(aux):                 # cuBLAS handle/workspace for aux outside capture
        torch.addmm(b, A[:C], W, out=out[:C])
    with torch.cuda.stream(main_s):
        torch.addmm(b, A[:C], W, out=out[:C])
    torch.cuda.synchronize()
    out.zero_()
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g, stream=main_s):
        bodies = (ctypes.c_void_p * K)()
        _lib.call("gns_graph_switch_begin", _lib.stream_ptr(main_s), n_dev.data_ptr(), C, K, bodies)
        for k in range(K):
            _lib.call("gns_graph_body_capture_begin", _lib.stream_ptr(aux), bodies[k])
            if k:
                rows = min(k * C, R)
                with torch.cuda.stream(aux):
                    torch.addmm(b, A[:rows], W, out=out[:rows])
            _lib.call("gns_graph_body_capture_end", _lib.stream_ptr(aux))
    ex = ctypes.c_void_p()
    _lib.call("gns_graph_instantiate", g.raw_cuda_graph(), 0, ctypes.byref(ex))
    ref = torch.addmm(b, A, W)
    for n in (0, 1, 8192, 8193, 100000, 138000, 176000):
        out.zero_()
        n_dev.fill_(n)
        torch.cuda.synchronize()
        _lib.call("gns_graph_launch", ex, _lib.stream_ptr(main_s))
        torch.cuda.synchronize()
        rows = min(-(-n // C) * C, R)
        ok = torch.allclose(out[:rows], ref[:rows], rtol=1e-2, atol=1e-2) and bool((out[rows:] == 0).all())
        print(f"n={n:6d}: rows computed {rows:6d} ok={ok}", flush=True)
    # timing: full capacity vs 138K rows
    for n in (176000, 138000):
        n_dev.fill_(n)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(main_s)
        for _ in range(50):
            _lib.call("gns_graph_launch", ex, _lib.stream_ptr(main_s))
        e.record(main_s)
        e.synchronize()
        print(f"n={n}: {s.elapsed_time(e) / 50 * 1e3:.1f} us per replay", flush=True)


if __name__ == "__main__":
    main()

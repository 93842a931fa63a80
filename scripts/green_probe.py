"""Do CUDA graphs captured on a green-context stream keep the SM partition?
A bandwidth-bound copy timed eagerly and as a graph replay on a 16-SM green
context stream vs the default stream; plus a libgns kernel (gather) on it.

    python scripts/green_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timeit(fn, stream, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(reps):
        fn()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    from torch.cuda.green_contexts import GreenContext
    from paper_2106_06150_b200 import _lib
    a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    main_s = torch.cuda.Stream()
    gc = GreenContext.create(16, 0)
    gs = gc.Stream()
    print("green stream", gs, flush=True)
    for name, st in (("primary stream", main_s), ("green 16-SM stream", gs)):
        with torch.cuda.stream(st):
            t_eager = timeit(lambda: b.copy_(a), st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                b.copy_(a)
            t_graph = timeit(g.replay, st)
            # a libgns kernel launched through the C ABI on this stream
            tab = torch.randn(1 << 20, 128, device="cuda")
            ids = torch.randint(0, 1 << 20, (200000,), device="cuda", dtype=torch.int32)
            out = torch.empty(200000, 128, device="cuda")

            def gather():
                _lib.call("gns_gather_rows", tab.data_ptr(), 128, 0, ids.data_ptr(), None, 200000, 128,
                          out.data_ptr(), 128, 0, _lib.stream_ptr(st))
            t_lib = timeit(gather, st)
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=st):
                gather()
            t_lib_graph = timeit(g2.replay, st)
        print(f"{name}: copy eager {t_eager:.1f} us, copy graph {t_graph:.1f} us, "
              f"gather eager {t_lib:.1f} us, gather graph {t_lib_graph:.1f} us", flush=True)


if __name__ == "__main__":
    main()

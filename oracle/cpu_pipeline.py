"""Reference-architecture CPU pipeline for the baseline timings — TEST/BENCH
INFRASTRUCTURE ONLY (``bench.py``'s cpu_baseline leg and ``--impl reference``).

Restates ``pool.py:69-193`` (fork workers build mini-batches from per-batch
``default_rng([seed, 32, epoch, index])`` streams, ordered delivery) feeding the
trainer loop body ``model.py:279-285`` (forward, loss, backward-with-recompute,
Adam) in float64 numpy/scipy — i.e. the reference's own CPU algorithm and RNG
cost, run on the box's host cores.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import gns as O
from . import model as OM

_STATE = {}


def _init(g, cache, cfg):
    _STATE["g"], _STATE["cache"], _STATE["cfg"] = g, cache, cfg


def _build(job):
    epoch, index, targets = job
    g, cache, cfg = _STATE["g"], _STATE["cache"], _STATE["cfg"]
    rng = np.random.default_rng([cfg.seed, 32, epoch, index])          # pool.py:70
    t0 = time.perf_counter()
    mb = O.build_minibatch(g, cache if cfg.strategy == "GNS" else None, targets, cfg, O.NumpyStream(rng))
    return index, mb, (time.perf_counter() - t0) * 1e3


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run(g, cache, cfg, dims, batches, epoch=0, workers=None, warmup=1, lr=0.003):
    """Time ``len(batches) - warmup`` reference steps (sample+gather+train).

    Returns dict(value=mb/s, steps, seconds, sample_ms, train_ms, workers)."""
    workers = max(1, (host_cores() - 1) if workers is None else workers)
    params = OM.init_params(dims, seed=0)
    state = OM.OAdam.zeros_like(params)
    jobs = [(epoch, i, t) for i, t in enumerate(batches)]
    ctx = mp.get_context("fork")
    train_ms, sample_ms = [], []
    with ctx.Pool(workers, initializer=_init, initargs=(g, cache, cfg)) as pool:
        it = pool.imap(_build, jobs, chunksize=1)
        t_start = None
        for j, (index, mb, s_ms) in enumerate(it):
            if j == warmup:
                t_start = time.perf_counter()
            t0 = time.perf_counter()
            OM.train_step(mb, g.features, g.labels, params, state, lr=lr)
            if j >= warmup:
                train_ms.append((time.perf_counter() - t0) * 1e3)
                sample_ms.append(s_ms)
        t_end = time.perf_counter()
    steps = len(batches) - warmup
    sec = t_end - t_start if t_start is not None else float("nan")
    return dict(value=steps / sec, steps=steps, seconds=sec, workers=workers,
                sample_ms=float(np.mean(sample_ms)) if sample_ms else 0.0,
                train_ms=float(np.mean(train_ms)) if train_ms else 0.0)

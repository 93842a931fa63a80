"""CPU oracle for the GNS hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the algorithm of the reference package
``gnsbench`` (``/root/reference/pkg/src/gnsbench``) for the hot path named in
``BASELINE.json:north_star``: the degree-proportional cache draw and its
induced cached-neighbor CSR, the NS/GNS per-layer neighbor samplers with
their importance weights, frontier dedup/relabel, the input-feature gather,
the weighted mean-aggregation SpMM and the float64 GraphSAGE trainer.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import it, and only as the checker (or the timed CPU
baseline).  The product path in ``paper_2106_06150_b200`` never imports it.

Randomness: the reference draws from numpy ``PCG64`` streams; the B200 build
uses counter-based Philox4x32-10 keyed on (seed, epoch, batch, layer, phase,
node, position).  The oracle restates the reference with the build's Philox
keys injected through the reference's own duck-typed ``rng.random(n)`` hook
(``sampling.py:166,214,233``).  It is pinned against the reference itself by
replaying the oracle's key arrays into ``gnsbench.build_minibatch``
(``tests/test_oracle.py::test_oracle_numpy_stream_equals_reference``) and by golden fixtures generated from the
reference (``tests/golden/make_golden.py``).
"""

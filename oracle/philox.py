"""Philox4x32-10 counter-based RNG and the GNS key layout (numpy, integer-exact).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

This is the RNG contract shared bit-for-bit with ``paper_2106_06150_b200/csrc/
gns_common.cuh``.  Philox4x32-10 is the Salmon et al. (SC'11) generator; its
known-answer vectors (Random123 ``kat_vectors``) are checked in
``tests/test_oracle.py::test_philox_kat``.

Key layout (restates the SPEC intent "deterministic per (seed, epoch,
batch_index, layer, dst node id)", ``SPEC.md:292``; the reference's
``pool.py:30-33`` stream tags are reused as the ``tag`` field):

    key     = (seed mod 2^32, epoch mod 2^32)
    counter = (pos >> 1, node, (tag << 24) | (layer << 16) | (phase << 8), batch)

One Philox block yields two 64-bit words; position ``pos`` takes word
``pos & 1``: ``x = (w[2j] << 32) | w[2j+1]`` and the 53-bit key is ``x >> 11``.
The float uniform handed to the reference is ``key53 * 2**-53`` — exactly how
numpy's ``Generator.random`` builds a double from 64 random bits, so the
reference's ``lexsort`` on the float keys orders exactly like the build's
integer comparison of ``(key53, pos)``.
"""

from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)

TAG_SHUFFLE = 31   # pool.py:30 _SHUFFLE
TAG_BATCH = 32     # pool.py:31 _BATCH
TAG_CACHE = 33     # pool.py:32 _CACHE
PHASE_CACHED = 0   # sampling.py:214 cached-phase draw
PHASE_FILL = 1     # sampling.py:233 fill-phase draw
PHASE_UNIFORM = 2  # sampling.py:166 NS draw


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10. All inputs broadcast; returns 4 uint64 arrays
    holding 32-bit words."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = (a.copy() for a in (c0, c1, c2, c3))
    for r in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
        if r < 9:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
    return c0, c1, c2, c3


def stream_word(tag: int, layer: int = 0, phase: int = 0) -> int:
    return ((tag & 0xFF) << 24) | ((layer & 0xFF) << 16) | ((phase & 0xFF) << 8)


def key53(seed, epoch, node, stream, batch, pos):
    """53-bit integer keys (uint64 array) for the given positions."""
    pos = np.asarray(pos, dtype=np.uint64)
    w0, w1, w2, w3 = philox4x32_10(pos >> np.uint64(1), node, stream, batch,
                                   seed, epoch)
    odd = (pos & np.uint64(1)).astype(bool)
    hi = np.where(odd, w2, w0)
    lo = np.where(odd, w3, w1)
    return ((hi << np.uint64(32)) | lo) >> np.uint64(11)


def uniform(seed, epoch, node, stream, batch, pos):
    """float64 uniforms in [0, 1): key53 * 2^-53 (exact)."""
    return key53(seed, epoch, node, stream, batch, pos).astype(np.float64) \
        * (1.0 / 9007199254740992.0)


# ---------------------------------------------------------------------------
# Feistel permutation for the epoch shuffle (pool.py:60-66 restated).
# ---------------------------------------------------------------------------

def _feistel_bits(n: int) -> int:
    bits = max(2, int(n - 1).bit_length())
    return bits + (bits & 1)


def feistel_permute(idx, n: int, seed: int, epoch: int):
    """Bijection of [0, n): balanced 4-round Feistel over 2h bits with cycle
    walking.  Round function = Philox word 0 of counter (x, round, tag31, 0)."""
    idx = np.asarray(idx, dtype=np.uint64)
    if n <= 1:
        return idx.copy()
    bits = _feistel_bits(n)
    h = bits // 2
    hmask = np.uint64((1 << h) - 1)
    stream = stream_word(TAG_SHUFFLE)

    def once(x):
        left = x >> np.uint64(h)
        right = x & hmask
        for r in range(4):
            f = philox4x32_10(right, r, stream, 0, seed, epoch)[0] & hmask
            left, right = right, left ^ f
        return (left << np.uint64(h)) | right

    y = once(idx)
    bad = y >= np.uint64(n)
    while bad.any():
        y[bad] = once(y[bad])
        bad = y >= np.uint64(n)
    return y

"""Numpy restatement of the reference graph-core ops (TEST INFRASTRUCTURE ONLY).

Each function names the reference lines it restates.  Results are plain numpy
arrays so the checker never depends on the product's types.  Pinned against the
reference ``graphs.py`` by ``tests/test_oracle_graphs.py`` (live import when
``/root/reference`` exists) and by the golden hashes in ``tests/golden``.
"""

from __future__ import annotations

import math

import numpy as np

UNREACHED = 0xFFFFFFFF  # graphs.py:13-17 (VID = uint32, UNREACHED = max VID)
DEFAULT_PROBS = (0.57, 0.19, 0.19, 0.05)  # graphs.py:21
PCG64_MULT = 0x2360ED051FC65DA44385DF649FCCF645  # numpy PCG64 (XSL-RR, 128-bit LCG)


def rmat_thresholds(probs=DEFAULT_PROBS):
    """The three Bernoulli thresholds of graphs.py:273-275, computed in the same
    float64 arithmetic, plus their exact integer form on the 53-bit draw
    ``k = next64 >> 11``: ``U < p  <=>  k < ceil(p * 2**53)`` (U = k * 2**-53 is
    exact and so is p * 2**53)."""
    a, b, c, d = (float(x) for x in probs)
    p_bottom = c + d
    p_right_top = b / (a + b)
    p_right_bottom = d / (c + d)
    ints = tuple(int(math.ceil(p * 2.0 ** 53)) for p in (p_bottom, p_right_top, p_right_bottom))
    return (p_bottom, p_right_top, p_right_bottom), ints


def check_rmat_args(scale, edge_factor, probs):
    """Argument checks of graphs.py:261-267."""
    if scale < 1 or edge_factor < 1:
        raise ValueError("scale and edge_factor must be >= 1")
    if (1 << scale) - 1 > UNREACHED:
        raise ValueError(f"scale {scale} overflows the vertex-id range")
    if min(probs) < 0 or abs(sum(probs) - 1.0) > 1e-9:
        raise ValueError("quadrant probabilities must be non-negative and sum to 1")


def generate_rmat(scale, edge_factor, seed, probs=DEFAULT_PROBS):
    """graphs.py:254-285.  Draw layout: for bit = scale-1 .. 0 the generator
    emits m source-bit uniforms then m destination-bit uniforms, so the draw
    index of (bit iteration k from the MSB, j in {0: src, 1: dst}, edge e) is
    (2k + j) * m + e.  Returns uint32 array (m, 2)."""
    check_rmat_args(scale, edge_factor, probs)
    m = edge_factor << scale
    (p_bottom, p_rt, p_rb), _ = rmat_thresholds(probs)
    rng = np.random.default_rng(seed)
    out = np.zeros((m, 2), dtype=np.uint32)
    for bit in reversed(range(scale)):
        lower_half = rng.random(m) < p_bottom
        right = rng.random(m) < np.where(lower_half, p_rb, p_rt)
        out[:, 0] |= lower_half.astype(np.uint32) << np.uint32(bit)
        out[:, 1] |= right.astype(np.uint32) << np.uint32(bit)
    return out


def pcg64_state_after(seed, draws):
    """Host model of the device generator's jump-ahead: (state, inc) of
    ``default_rng(seed)`` after ``draws`` outputs, via numpy's own advance()."""
    bg = np.random.PCG64(seed)
    bg.advance(draws)
    st = bg.state["state"]
    return st["state"], st["inc"]


def pcg64_draw(seed, index):
    """The index-th float64 uniform of default_rng(seed) (0-based)."""
    bg = np.random.PCG64(seed)
    bg.advance(index)
    return np.random.Generator(bg).random()


def symmetrize(edges, num_vertices):
    """graphs.py:218-230: drop self-loops, add mirrors, dedup, sort by (src,dst).
    Restated with a (src << 32 | dst) key, which sorts identically to the
    reference's src * n + dst key."""
    e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
    if e.shape[0] == 0 or num_vertices == 0:
        return np.empty((0, 2), dtype=np.uint32)
    s = e[:, 0].astype(np.uint64)
    t = e[:, 1].astype(np.uint64)
    keep = s != t
    s, t = s[keep], t[keep]
    keys = np.concatenate([(s << np.uint64(32)) | t, (t << np.uint64(32)) | s])
    keys.sort()
    if keys.size:
        first = np.ones(keys.size, dtype=bool)
        first[1:] = keys[1:] != keys[:-1]
        keys = keys[first]
    out = np.empty((keys.size, 2), dtype=np.uint32)
    out[:, 0] = (keys >> np.uint64(32)).astype(np.uint32)
    out[:, 1] = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return out


def build_csr(edges, num_vertices):
    """graphs.py:233-251: validate a symmetrized edge list and build CSR.
    Returns (offsets int64[n+1], adjacency uint32[m]).  Raises ValueError with
    the reference's messages on self-edge / duplicate / missing reverse."""
    e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
    n = int(num_vertices)
    s = e[:, 0].astype(np.uint64)
    t = e[:, 1].astype(np.uint64)
    if e.shape[0]:
        if np.any(s == t):
            raise ValueError("input is not symmetrized: self-edge present")
        fwd = np.sort((s << np.uint64(32)) | t)
        if fwd.size > 1 and np.any(fwd[1:] == fwd[:-1]):
            raise ValueError("input is not symmetrized: duplicate edge present")
        rev = np.sort((t << np.uint64(32)) | s)
        if not np.array_equal(fwd, rev):
            raise ValueError("input is not symmetrized: missing reverse edge")
        # rows in (src, dst) order == the reference's lexsort((dst, src))
        adjacency = (fwd & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    else:
        adjacency = np.empty(0, dtype=np.uint32)
    counts = np.bincount(e[:, 0], minlength=n) if e.shape[0] else np.zeros(n, dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts, dtype=np.int64)]).astype(np.int64)
    return offsets, adjacency


def partition_1d(offsets, num_parts):
    """graphs.py:288-305: boundary k = first vertex whose cumulative degree
    reaches round-half-up(|E| k / P) (searchsorted 'left' on offsets)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    n = offsets.size - 1
    m = int(offsets[-1]) if offsets.size else 0
    if num_parts < 1:
        raise ValueError("num_parts must be >= 1")
    if n and num_parts > n:
        raise ValueError("num_parts exceeds the number of vertices")
    b = np.empty(num_parts + 1, dtype=np.int64)
    b[0] = 0
    b[num_parts] = n
    for k in range(1, num_parts):
        target = (2 * m * k + num_parts) // (2 * num_parts)
        b[k] = np.searchsorted(offsets, target, side="left")
    return b


def sample_roots(offsets, count=64, seed=2103):
    """Root protocol of BASELINE.md §2 / SURVEY §8(d): ``count`` distinct
    non-isolated roots, ``default_rng(seed).choice(flatnonzero(deg>0), count,
    replace=False)``."""
    deg = np.diff(np.asarray(offsets, dtype=np.int64))
    nz = np.flatnonzero(deg > 0)
    k = min(count, nz.size)
    return nz[np.random.default_rng(seed).choice(nz.size, k, replace=False)].astype(np.int64)

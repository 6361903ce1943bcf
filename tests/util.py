"""Test helpers: hashes and small hand-made graphs (SPEC example shapes)."""

import hashlib

import numpy as np

from oracle import graphs as og


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def csr_of_undirected(n, pairs):
    """Symmetrized CSR (oracle) of an undirected edge list."""
    e = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
    return og.build_csr(og.symmetrize(e, n), n)


def path_graph(n):
    return csr_of_undirected(n, [(i, i + 1) for i in range(n - 1)])


def star_graph(leaves):
    return csr_of_undirected(leaves + 1, [(0, i) for i in range(1, leaves + 1)])


def components_graph(k=5, size=40, seed=3):
    rng = np.random.default_rng(seed)
    pairs = []
    for c in range(k):
        base = c * size
        for i in range(1, size):
            pairs.append((base + i, base + int(rng.integers(0, i))))
    return csr_of_undirected(k * size, pairs)


def gnp_graph(n, p, seed=7):
    rng = np.random.default_rng(seed)
    m = rng.binomial(n * (n - 1) // 2, p)
    s = rng.integers(0, n, m)
    t = rng.integers(0, n, m)
    return csr_of_undirected(n, np.stack([s, t], 1))


def rmat_graph(scale, ef=8, seed=1):
    raw = og.generate_rmat(scale, ef, seed)
    return og.build_csr(og.symmetrize(raw, 1 << scale), 1 << scale)

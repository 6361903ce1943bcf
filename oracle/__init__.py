"""CPU oracle for the ButterFly BFS hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference's algorithm for the path
that the CUDA library implements:

* ``oracle.graphs``   -- graph-core ops of ``pkg/src/bflybfs/graphs.py``
  (RMAT generator, symmetrize, build_csr, partition_1d), restated.
* ``oracle.bfs``      -- the bfs-oracle module (``SPEC.md:122-176``,
  Alg. 1 ``PAPER.md:100-138``): ``bfs_top_down`` / ``frontier_sizes``.
* ``oracle.cbfs``     -- the same top-down BFS restated in C + OpenMP
  (``bfs_omp.c``, all host threads: the paper's OpenMP worker model,
  ``PAPER.md:585``); bench.py's timed CPU baseline and reference arm.
* ``oracle.schedule`` -- the butterfly-schedule module (``SPEC.md:178-265``).
* ``oracle.engine``   -- the lockstep multi-node engine (``SPEC.md:267-367``,
  Alg. 2 ``PAPER.md:279-374``) with ``RunStats`` accounting.
* ``oracle.validate`` -- DistanceArray / parent certificates
  (``SPEC.md:130-132``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2103_13577_b200`` never
imports it; the product path has no CPU fallback.

Parity pinning: the reference ships no BFS code, only ``graphs.py``.  The
graph ops here are pinned against the reference ``graphs.py`` itself (imported
from ``/root/reference/pkg/src`` when present, and via the committed golden
hashes in ``tests/golden/`` made by ``tests/golden/make_golden.py``).  The BFS
levels are pinned against an independent BFS (``scipy.sparse.csgraph``) in the
golden script; BFS levels are mathematically unique, so any correct BFS
matches bit-exactly.
"""

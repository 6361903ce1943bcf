"""B200-native ButterFly BFS (arXiv 2103.13577).

Drop-in for the reference package ``bflybfs``'s hot path: ``graphs`` (device
generator / symmetrize / CSR / partition), ``schedule`` (butterfly
schedule), ``engine.run`` (multi-node top-down BFS with butterfly frontier
synchronization) over hand-written sm_100a kernels in ``libbflybfs.so``.
"""

from . import _lib

__version__ = "0.1.0"
__all__ = ["graphs", "schedule", "engine", "device", "_lib"]

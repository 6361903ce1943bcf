"""Developer tool: device time of one BFS on deep graphs (paths) with the
thin-level / sparse paths on and off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_13577_b200.device import DeviceGraph  # noqa: E402

for n in (50000, 200000, 1000000):
    i = np.arange(n - 1, dtype=np.int64)
    src = np.concatenate([i, i + 1])
    dst = np.concatenate([i + 1, i])
    o = np.argsort(src * n + dst, kind="stable")
    src, dst = src[o], dst[o]
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off)
    dg = DeviceGraph.from_csr(off, dst.astype(np.uint32))
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=True)
    for sparse in (True, False):
        dg.set_sparse_levels(sparse)
        dg.bfs(0, levels=False)
        _, _, _, st, _ = dg.bfs(0, levels=False, max_levels=n + 1)
        print(f"path({n}) from an end: {st.levels} levels, thin/sparse={'on' if sparse else 'off'}: "
              f"{st.elapsed_ms:.1f} ms device, {1e3 * st.elapsed_ms / st.levels:.2f} us/level, "
              f"{st.kernel_launches} launches", flush=True)

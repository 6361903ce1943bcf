import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libbflybfs.so on cuda:0)")
    config.addinivalue_line("markers", "slow: larger-scale GPU parity / property checks")
    lib = os.path.join(ROOT, "paper_2103_13577_b200", "libbflybfs.so")
    if not os.path.exists(lib):  # the driver runs build() first; this is a fallback
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2103_13577_b200", "csrc"), "-j8"],
                       check=True, stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def s10():
    z = np.load(os.path.join(GOLDEN_DIR, "s10_ef8.npz"))
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def reference_graphs():
    """The reference graphs.py, importable only where /root/reference exists."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference sources not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from bflybfs import graphs

    return graphs


@pytest.fixture(scope="session")
def reference_objects():
    """Reference Graph / Partition objects for the drop-in tests, never
    skipped: the live reference's own objects where /root/reference exists,
    otherwise foreign stand-in objects (tests/ref_types.py) over arrays the
    reference produced (tests/golden/ref_objects.npz).  Returns a loader
    name -> (Graph, Partition, {root: levels}, source)."""
    from tests import ref_types

    def load(name):
        g, p, levels = ref_types.load(name)
        if os.path.isdir(REF_SRC):
            if REF_SRC not in sys.path:
                sys.path.insert(0, REF_SRC)
            from bflybfs import graphs as R

            s, ef, seed = {"s12_ef8_seed3": (12, 8, 3), "s10_ef8_seed1": (10, 8, 1)}[name]
            rg = R.build_csr(R.symmetrize(R.generate_rmat(s, ef, seed)))
            rp = R.partition_1d(rg, p.num_parts)
            assert np.array_equal(rg.offsets, g.offsets) and np.array_equal(rg.adjacency, g.adjacency)
            assert np.array_equal(rp.boundaries, p.boundaries)
            return rg, rp, levels, "live reference"
        return g, p, levels, "reference arrays (fixture)"

    return load

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")

# the reference's own test modules (vendored verbatim, tools/vendor_reference_tests.sh)
# import `hvbem`: they run in a subprocess behind the import alias
# (tests/test_reference_suite.py), never in this session
collect_ignore = ["reference_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhvb.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def _cfg3_parts(F, level_sph, level_encl):
    v1, t1 = F.sphere_mesh_parts(level_sph, radius=0.5, center=(-0.6, 0.0, 0.0), tag=0)
    v2, t2 = F.sphere_mesh_parts(level_sph, radius=0.5, center=(0.6, 0.0, 0.0), tag=1, id_offset=len(v1))
    v3, t3 = F.sphere_mesh_parts(level_encl, radius=3.0, flip=True, tag=2, id_offset=len(v1) + len(v2))
    return np.vstack([v1, v2, v3]), t1 + t2 + t3


def build_case(name):
    """The golden-fixture input meshes, built with OUR generators (which are
    bit-identical to the reference's, see test_mesh_parity)."""
    from paper_2003_12663_b200 import fixtures as F
    from paper_2003_12663_b200.mesh import EPS0

    if name == "sphere2":
        return F.sphere_mesh(2)
    if name == "cap2":
        return F.concentric_mesh(2, [(0.5, "electrode 1.0"), (1.0, "electrode 0.0")])
    if name == "floatshell1":
        return F.concentric_mesh(1, [(0.5, "electrode 1.0"), (0.75, f"sheet 0 {EPS0!r} {EPS0!r}"),
                                     (1.0, "electrode 0.0")])
    if name in ("diel1", "diel2"):
        return F.concentric_mesh(int(name[-1]), [(0.5, "electrode 1.0"),
                                                 (0.75, f"dielectric {EPS0!r} {2 * EPS0!r}"),
                                                 (1.0, "electrode 0.0")])
    if name == "gap2":
        return F.concentric_mesh(2, [(1.0, "electrode 1.0"), (1.02, "electrode 0.0")])
    if name == "cfg3mini":
        v, tris = _cfg3_parts(F, 1, 0)
        ids = np.array([t[0] for t in tris])
        tags = np.array([t[1] for t in tris])
        return F.mesh_from_parts(v, ids, tags, ["patch 0 electrode 1.0", "patch 1 floating 0",
                                               "patch 2 electrode 0.0"])
    if name == "plates":
        pa, ta = F._box_grid((0.2, 0.2, 0.01), (6, 6, 1))
        pb, tb = F._box_grid((0.2, 0.2, 0.01), (6, 6, 1))
        pb = pb + np.array([0.013, 0.0, 0.024])
        ids = np.vstack([ta, tb + len(pa)])
        tags = np.concatenate([np.zeros(len(ta), int), np.ones(len(tb), int)])
        return F.mesh_from_parts(np.vstack([pa, pb]), ids, tags, ["patch 0 electrode 1.0",
                                                                  "patch 1 electrode -1.0"])
    if name == "rodmini":
        return F.rod_plane_mesh(0.12)
    raise KeyError(name)


CASES = ["sphere2", "cap2", "floatshell1", "diel1", "diel2", "gap2", "cfg3mini", "plates", "rodmini"]


@pytest.fixture(scope="session")
def cases():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = build_case(name)
        return cache[name]

    return get


def gpu_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False

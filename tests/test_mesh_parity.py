"""Our vectorised mesh construction and fixture generators reproduce the
reference's input arrays bit for bit (hashes recorded by make_golden.py)."""

import hashlib

import numpy as np
import pytest

from conftest import CASES
from paper_2003_12663_b200 import fixtures as F


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("level", [1, 2, 3, 4])
def test_sphere_ladder_bitwise(golden, level):
    m = F.sphere_mesh(level)
    assert h(m.vertices) == str(golden[f"sphere{level}_vertices_sha"])
    assert h(m.circumcenters) == str(golden[f"sphere{level}_cc_sha"])
    assert h(m.circumradii) == str(golden[f"sphere{level}_cr_sha"])


@pytest.mark.parametrize("name", CASES)
def test_case_meshes(golden, cases, name):
    m = cases(name)
    p = name + "_mesh_"
    assert h(m.vertices) == str(golden[p + "vertices_sha"])
    assert h(m.circumcenters) == str(golden[p + "cc_sha"])
    assert h(m.circumradii) == str(golden[p + "cr_sha"])
    np.testing.assert_allclose(m.lumped_weights, golden[p + "weights"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(m.colloc_normals, golden[p + "normals"], rtol=0, atol=1e-13)
    rhs = golden[name + "_rhs"]
    assert len(rhs) == m.n_collocation + m.n_floating

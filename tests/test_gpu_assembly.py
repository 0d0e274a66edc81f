"""stencil assembly on the device (mpk_stencil_assemble) is
bit-identical to generate_stencil's (which is pinned to the reference by
SHA-256, tests/golden/stencils.json), up to the BASELINE sizes."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2105_07544_b200 as mk

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stencils.json")))


@pytest.mark.parametrize("preset,nx", [("Laplace2D", 17), ("Laplace3D", 9), ("UniFlow2D", 33), ("BentPipe2D", 48),
                                       ("Stretched2D", 21), ("Laplace3D", 2), ("BentPipe2D", 2)])
def test_device_assembly_bit_identical(cuda, preset, nx):
    spec = mk.ProblemSpec(preset, nx)
    h = mk.generate_stencil(spec)
    d = mk.generate_stencil(spec, on_device=True)
    assert d.nnz == h.nnz and d.n == h.n
    assert np.array_equal(d.row_ptr, h.row_ptr)
    assert np.array_equal(d.col_idx, h.col_idx)
    assert np.array_equal(d.values.view(np.uint64), h.values.view(np.uint64))
    x = np.random.default_rng(1).standard_normal(h.n)
    d.use_stencil = False
    assert np.array_equal(mk.spmv(d, x), mk.spmv(h, x))   # the kept device copy is the CSR


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("preset,nx", [("BentPipe2D", 1500), ("Laplace3D", 200)])
def test_device_assembly_baseline_sizes(cuda, preset, nx):
    spec = mk.ProblemSpec(preset, nx)
    d = mk.generate_stencil(spec, on_device=True)
    h = mk.generate_stencil(spec)
    assert np.array_equal(d.row_ptr, h.row_ptr) and np.array_equal(d.col_idx, h.col_idx)
    assert np.array_equal(d.values.view(np.uint64), h.values.view(np.uint64))
    g = GOLD["%s_%d" % (preset, nx)]   # the reference's own arrays (make_golden.py)
    assert _sha(d.row_ptr) == g["row_ptr"] and _sha(d.col_idx) == g["col_idx"] and _sha(d.values) == g["values"]

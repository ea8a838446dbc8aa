"""CPU checks of the oracle-side input generator and sample meshes (no GPU).

The bench's reference arm and the CPU half of tools/full_step_parity.py build their
inputs with the oracle's restatement of the frozen generator
so that those processes never load the product library.  The two generators must give
bit-identical values; the reference arm's z-slabs must be cells of the full mesh.
"""
import numpy as np
import pytest


def test_oracle_uniform_matches_product_bitwise(ref):
    import paper_2107_07776_b200 as dg
    for seed, n in ((0, 1), (1002, 4097), (2002, 10000)):
        assert np.array_equal(ref.seeded_uniform(seed, n), dg.seeded_uniform(seed, n))
    assert np.array_equal(ref.seeded_uniform(5, 100, 0.5, 2.0), dg.seeded_uniform(5, 100, 0.5, 2.0))


@pytest.mark.parametrize("dim,seed,scale", [(2, 0, 1.0), (3, 1, 1.0), (3, 2, 1.0), (3, 4, 0.37)])
def test_oracle_synth_field_matches_product_bitwise(ref, dim, seed, scale):
    import paper_2107_07776_b200 as dg
    f, g = ref.SynthField(dim, seed, scale), dg.SynthField(dim, seed, scale)
    assert np.array_equal(f.user, g.user)
    rng = np.random.default_rng(seed)
    for _ in range(50):
        x = rng.random(dim)
        assert np.array_equal(f.eval(x), g.eval(x))


def test_oracle_interpolation_threads_agree(ref):
    R = ref.RefCtx(3, 4, 3, 2)
    f = ref.SynthField(3, 2)
    a, b = f.interpolate(R, 1), f.interpolate(R, 3)
    assert np.array_equal(a, b)
    # FunctionSpace::interpolate nodes: the value at a node is the field at that node
    xn = np.zeros((R.ncells, 64, 3))
    ref.lib().ref_node_points(R.h, 0, ref.P(xn))
    cell, j = 17, 21
    v = f.eval(xn[cell, j])
    assert np.array_equal(a.reshape(R.ncells, 3, 64)[cell, :, j], v)


def test_slab_cells_are_cells_of_the_full_mesh(ref):
    n, z0, nz = 6, 2, 3
    full = ref.RefCtx(3, n, 2, 1)
    slab = ref.RefCtx.slab(n, z0, nz, 2, 1)
    assert slab.ncells == n * n * nz
    assert slab.n_boundary == 2 * 2 * n * nz + 2 * n * n
    assert slab.n_interior == 2 * (n - 1) * n * nz + n * n * (nz - 1)
    xf, xs = full.cell_vertices(), slab.cell_vertices()
    c0 = z0 * n * n
    assert np.array_equal(xs, xf[c0:c0 + n * n * nz])
    # same cells, same inputs -> the reference's slab apply equals the full apply on
    # every cell whose z-neighbours are inside the slab (interior faces identical)
    f = ref.SynthField(3, 2)
    w_full, w_slab = f.interpolate(full), f.interpolate(slab)
    nb = 3 * 27
    assert np.array_equal(w_slab, w_full[c0 * nb:(c0 + n * n * nz) * nb])
    x = ref.seeded_uniform(1002, full.n_u)
    coefs = (3.7, 0.01, 0.5, 0.0)
    yf = full.momentum(coefs, w_full, x)
    ys = slab.momentum(coefs, w_slab, x[c0 * nb:(c0 + n * n * nz) * nb])
    mid = slice((c0 + n * n) * nb, (c0 + 2 * n * n) * nb)  # the slab's middle layer
    np.testing.assert_allclose(ys[n * n * nb:2 * n * n * nb], yf[mid], rtol=0, atol=1e-12 * np.abs(yf).max())


def test_reference_kern_is_the_avx2_backend(ref):
    """ref_kern drives kern:: (kernels.hpp:34-43); on an AVX2 host axpy is one FMA per
    element (kernels_avx2.cpp:12-20), which the device kernel reproduces bit for bit."""
    from fractions import Fraction
    x = ref.seeded_uniform(1, 257)
    y = ref.seeded_uniform(2, 257)
    out = ref.kern("axpy", 0.37, x, y)
    if ref.lib().ref_backend().decode() == "avx2":
        fma = [float(Fraction(0.37) * Fraction(a) + Fraction(b)) for a, b in zip(x, y)]
        assert np.array_equal(out, np.array(fma))
    assert ref.kern("max_abs_diff", 0.0, x, y) == np.abs(x - y).max()

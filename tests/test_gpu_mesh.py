"""GPU parity on the mesh / road class of the paper's Table I (PAPER.md:167-177:
hugetrace, venturiLevel3, *_osm, road_central): weighted grid Laplacians with
dropped edges (synthgen.grid_laplacian, recipe C6/C6S in DESIGN.md). Low, uniform
degree (0..5 entries per row, isolated vertices are empty rows) puts every row in
the SELL-32 part of the SpMV format (no big rows), the opposite of R-MAT.
Tolerances as tests/test_gpu_parity.py (north_star)."""
import numpy as np
import pytest

import oracle as O
import synthgen as S
from test_gpu_parity import TOL, T_all, check_solve, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_2201_07498_b200 as T
    return T


@pytest.fixture(scope="module")
def c6s():
    return S.config_matrix("C6S")


@pytest.mark.parametrize("G", [1, 3])
def test_layout_bit_exact_mesh(T, c6s, G):
    with T.TopkEig(c6s, 8, "f32", "f64", parts=G) as h:
        b = h.partition()
        assert np.array_equal(b, O.partition(c6s.rowptr, G))
        for g in range(G):
            rp, col, val, npad = h.layout(g)
            orp, ocol, oval, onpad = O.layout(c6s.rowptr, c6s.col, c6s.val, G, b, g, "f32")
            assert npad == onpad and np.array_equal(rp, orp)
            assert np.array_equal(col, ocol) and np.array_equal(val, oval)


@pytest.mark.parametrize("storage,G", [("f64", 1), ("f32", 1), ("f64", 2)])
def test_spmv_parity_mesh(T, c6s, storage, G):
    A = c6s
    assert (np.diff(A.rowptr) == 0).any()  # isolated vertices: empty rows
    x = np.random.default_rng(6).standard_normal(A.n)
    with T.TopkEig(A, 4, storage, "f64", parts=G) as h:
        y = h.debug_spmv(x)
    xr = x.astype(np.float32).astype(np.float64) if storage == "f32" else x
    av = A.val if storage == "f64" else A.val.astype(np.float32).astype(np.float64)
    yr = O.spmv(A.rowptr, A.col, av, xr)
    bound = (np.diff(A.rowptr) + 2) * 2.0 ** -53 * O.spmv(A.rowptr, A.col, np.abs(av), np.abs(xr))
    assert np.all(np.abs(y - yr) <= bound + 1e-300)


@pytest.mark.parametrize("K,m,storage", [(24, 24, "f32"), (24, 24, "f64"), (8, 64, "f32")])
def test_mesh_parity(T, c6s, K, m, storage):
    A = c6s
    ref = O.solve(A.rowptr, A.col, A.val, K=K, m=m, seed=6, tau=O.TAU["f64"])
    r = T.solve(A, K, storage=storage, compute="f64", m=m, seed=6)
    assert normwise(T_all(T, A, K, storage, "f64", m, 6), ref.theta_all) <= TOL[storage]
    check_solve(r, ref, TOL[storage])


def test_grid_dirichlet_closed_form_gpu(T):
    """GPU solve on the 2-D Dirichlet Laplacian from the P16 start vector: Ritz values
    equal the closed-form eigenvalues (pin P16 on the CUDA path)."""
    nx, ny = 300, 200
    A = S.grid_dirichlet(nx, ny)
    modes = [(1, 1), (300, 200), (40, 30), (260, 170), (100, 60), (200, 140), (150, 100), (120, 40)]
    x = np.arange(1, nx + 1)
    y = np.arange(1, ny + 1)
    v1 = np.zeros(nx * ny)
    for i, j in modes:
        v1 += np.outer(np.sin(np.pi * j * y / (ny + 1)), np.sin(np.pi * i * x / (nx + 1))).ravel()
    lam = np.sort([4 - 2 * np.cos(np.pi * i / (nx + 1)) - 2 * np.cos(np.pi * j / (ny + 1)) for i, j in modes])
    with T.TopkEig(A, 8, "f64", "f64", m=8) as h:
        h.solve(v1=v1, vectors=False)
        th = np.sort(h.tridiag()[2])
    assert np.abs(th - lam).max() <= 1e-11

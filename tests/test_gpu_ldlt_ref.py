"""f3 LDL^T against the REFERENCE'S OWN linalg.cpp (oracle/_ref, compiled
unmodified; its doctest suite test_linalg.cpp passes against that build).

The inertia of every native factorisation kernel (blocked panel, cluster
panel, one-cluster, cooperative grid) must equal the reference's, including the reference's
zero-pivot rules (linalg.cpp:143-157 negligible column -> exact zero pivot;
:226-229 |d| <= 1e-11 max|SAS| -> zero L column), which decide the inertia
of numerically rank-deficient KKT matrices -- the case the IPM's inertia
correction (ipm.cpp:520-557) exists for.  Plus the large-n paths: the
multi-CTA grid kernel (n ~ 4000) and the native grid kernel with iterative
refinement beyond 32768 rows (cuSOLVER only past the int32 bound, n > 46340).
"""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import ldlt_oracle as lo
from oracle import ref

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not shipped")


@pytest.fixture(autouse=True)
def _gpu():
    if not has_gpu():
        pytest.skip("no GPU")


def sym(rng, n):
    m = rng.uniform(-1, 1, (n, n))
    return 0.5 * (m + m.T)


def cases():
    rng = np.random.default_rng(7)
    out = {}
    out["identity"] = np.eye(3)
    out["diag"] = np.diag([2.0, -5.0])
    out["zero"] = np.zeros((5, 5))
    out["spectrum"] = lo.matrix_with_spectrum(rng, [4, 3, 2, 1, -1, -2, -3, 0])
    for n in (2, 17, 33, 65, 150):
        out[f"random_{n}"] = sym(rng, n)
    a = sym(rng, 90)
    a[np.diag_indices(90)] *= 1e-8
    out["heavy_pivoting"] = a
    b = rng.uniform(-1, 1, (20, 17))
    out["rank_deficient"] = b @ b.T
    # a well-conditioned block beside a block at noise level (1e-14 of the
    # scale): the reference takes zero pivots there instead of forming 2x2
    # blocks from noise
    r = sym(rng, 40) + 4 * np.eye(40)
    e = 1e-14 * sym(rng, 12)
    out["noise_block"] = np.block([[r, np.zeros((40, 12))], [np.zeros((12, 40)), e]])
    # KKT with linearly dependent constraint rows (+ noise): the zero
    # eigenvalues the inertia correction must see
    n, m = 60, 20
    H = sym(rng, n) + np.diag(rng.uniform(1, 3, n))
    J = rng.uniform(-1, 1, (m, n))
    J[10:] = J[:10] + 1e-15 * rng.uniform(-1, 1, (10, n))
    out["kkt_dependent_rows"] = np.block([[H, J.T], [J, np.zeros((m, m))]])
    # [[A, B], [B^T, B^T A^-1 B + E]] with E at 1e-13: rank n1 up to noise,
    # every row O(1) (Ruiz cannot scale the deficiency away), so the last
    # pivots are noise-level Schur-complement entries -- the reference takes
    # zero pivots there (linalg.cpp:143-157, 226-229) instead of 2x2 blocks
    A = sym(rng, 30) + 4 * np.eye(30)
    B = rng.uniform(-1, 1, (30, 6))
    S = B.T @ np.linalg.solve(A, B)
    out["schur_noise"] = np.block([[A, B], [B.T, 0.5 * (S + S.T) + 1e-13 * sym(rng, 6)]])
    return out


CASES = cases()


@needs_ref
@pytest.mark.parametrize("path", ["panel", "cpanel", "cluster", "grid"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_inertia_equals_reference_linalg(monkeypatch, path, name):
    import paper_2509_22462_b200 as gb
    monkeypatch.setenv("GBOPT_LDLT_KERNEL", path)
    A = CASES[name]
    want = ref.RefLdlt(A).inertia
    f = gb.ldlt_factor(A)
    assert f.inertia == want, (name, path, f.inertia, want)
    if want[2] == 0:
        b = np.linspace(-1, 1, A.shape[0])
        x = f.solve(b)
        xr = ref.RefLdlt(A).solve(b)
        assert np.abs(A @ x - b).max() <= 1e-9 * (np.abs(A).max() * np.abs(x).max() + 1.0)
        assert np.abs(x - xr).max() <= 1e-6 * (np.abs(xr).max() + 1.0)
    else:
        with pytest.raises(gb.SingularError):
            f.solve(np.ones(A.shape[0]))


@needs_ref
@pytest.mark.parametrize("path", ["", "grid"])
def test_n4000_matches_reference(monkeypatch, path):
    """n = 4000: the default path (the cluster-panel kernel, ldlt_bkq.cuh:
    2 rows per thread, compacting updates) and the grid kernel with several
    CTAs per SM and > 256 partial maxima."""
    import paper_2509_22462_b200 as gb
    if path:
        monkeypatch.setenv("GBOPT_LDLT_KERNEL", path)
    rng = np.random.default_rng(4000)
    n, m = 3200, 800
    H = sym(rng, n) + np.diag(10.0 ** rng.uniform(-2, 4, n))
    J = rng.uniform(-1, 1, (m, n))
    K = np.block([[H, J.T], [J, -1e-8 * np.eye(m)]])
    ref.set_threads(16)
    want = ref.RefLdlt(K).inertia
    f = gb.ldlt_factor(K)
    assert f.inertia == want
    b = rng.uniform(-1, 1, n + m)
    x = f.solve(b)
    assert np.abs(K @ x - b).max() <= 1e-8 * (np.abs(K).max() * np.abs(x).max() + 1.0)


def test_beyond_32768_rows_refined_solve():
    """n = 33000 (the native grid kernel since round 2; cuSOLVER before):
    the refinement residual covers every row (ldlt_residual_kernel strides
    over rows).  A
    saddle point [[D, J^T], [J, 0]] with D > 0 and J of full row rank has
    inertia (n1, m, 0) exactly."""
    import paper_2509_22462_b200 as gb
    rng = np.random.default_rng(33)
    n1, m = 32000, 1000
    K = np.zeros((n1 + m, n1 + m))
    K[np.arange(n1), np.arange(n1)] = rng.uniform(1.0, 4.0, n1)
    J = np.zeros((m, n1))
    for i in range(m):  # each constraint touches its own 32 variables (+ a shared one)
        J[i, 32 * i:32 * i + 32] = rng.uniform(0.5, 1.5, 32)
        J[i, n1 - 1 - i] += 1.0
    K[n1:, :n1] = J
    K[:n1, n1:] = J.T
    f = gb.ldlt_factor(K, keep_input=True)
    assert f.inertia == (n1, m, 0)
    b = rng.uniform(-1, 1, n1 + m)
    x = f.solve(b)
    r = K @ x - b
    assert np.abs(r).max() <= 1e-10 * (np.abs(K).max() * np.abs(x).max() + 1.0)
    assert np.abs(r[-(n1 + m - 32768):]).max() <= 1e-10 * (np.abs(x).max() + 1.0)


@needs_ref
@pytest.mark.parametrize("n1,m,seed", [(1800, 700, 1), (5200, 1800, 2), (7000, 2000, 3)])
def test_cluster_panel_saddle_point_matches_reference(monkeypatch, n1, m, seed):
    """The cluster-panel kernel on saddle-point KKT matrices [[H, J^T], [J, 0]]
    with an indefinite H: most pivots of the constraint block are 2x2 blocks
    or interchanges with far rows, so each panel displaces rows the next
    panel's compaction must carry (1, 2 and 3 rows per thread)."""
    import paper_2509_22462_b200 as gb
    monkeypatch.setenv("GBOPT_LDLT_KERNEL", "cpanel")
    rng = np.random.default_rng(seed)
    H = sym(rng, n1) + np.diag(rng.uniform(-3, 3, n1))
    J = rng.uniform(-1, 1, (m, n1))
    K = np.block([[H, J.T], [J, np.zeros((m, m))]])
    ref.set_threads(16)
    want = ref.RefLdlt(K).inertia
    f = gb.ldlt_factor(K)
    assert f.inertia == want
    b = rng.uniform(-1, 1, n1 + m)
    x = f.solve(b)
    assert np.abs(K @ x - b).max() <= 1e-8 * (np.abs(K).max() * np.abs(x).max() + 1.0)


def test_cluster_panel_four_rows_per_thread_known_inertia(monkeypatch):
    """n = 16000 through the cluster-panel kernel (forced): 4 rows per thread,
    nb limited by the slice, several hundred compacting updates.  A saddle
    point [[D, J^T], [J, 0]] with D > 0 and J of full row rank has inertia
    (n1, m, 0) exactly, and the refined solve must reach the residual bar."""
    import paper_2509_22462_b200 as gb
    monkeypatch.setenv("GBOPT_LDLT_KERNEL", "cpanel")
    rng = np.random.default_rng(16)
    n1, m = 15000, 1000
    K = np.zeros((n1 + m, n1 + m))
    K[np.arange(n1), np.arange(n1)] = rng.uniform(1.0, 4.0, n1)
    J = np.zeros((m, n1))
    for i in range(m):
        J[i, 15 * i:15 * i + 15] = rng.uniform(0.5, 1.5, 15)
        J[i, n1 - 1 - i] += 1.0
    K[n1:, :n1] = J
    K[:n1, n1:] = J.T
    f = gb.ldlt_factor(K)
    assert f.inertia == (n1, m, 0)
    b = rng.uniform(-1, 1, n1 + m)
    x = f.solve(b)
    assert np.abs(K @ x - b).max() <= 1e-10 * (np.abs(K).max() * np.abs(x).max() + 1.0)


@pytest.mark.parametrize("dim,kernel", [(2048, "panel"), (2049, "cpanel"), (8500, "cpanel"), (8501, "grid")])
def test_default_kernel_ranges_at_their_edges(dim, kernel):
    """The default factorisation kernel at the edges of its size ranges
    (one-CTA panel n <= 2048, cluster panel 2048 < n <= 8500, grid beyond;
    read from the GBOPT_LDLT_TIMING trace), each with the exact inertia of a
    saddle point [[D, J^T], [J, 0]] (D > 0, J of full row rank) and a refined
    solve at the residual bar.  Separate process: the trace goes to stderr."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2509_22462_b200 as gb\n"
        "dim = %d; m = dim // 10; n1 = dim - m\n"
        "rng = np.random.default_rng(dim)\n"
        "K = np.zeros((dim, dim))\n"
        "K[np.arange(n1), np.arange(n1)] = rng.uniform(1.0, 4.0, n1)\n"
        "for i in range(m):\n"
        "    K[n1 + i, 7 * i:7 * i + 7] = rng.uniform(0.5, 1.5, 7)\n"
        "    K[n1 + i, n1 - 1 - i] += 1.0\n"
        "K[:n1, n1:] = K[n1:, :n1].T\n"
        "f = gb.ldlt_factor(K)\n"
        "b = rng.uniform(-1, 1, dim); x = f.solve(b)\n"
        "res = np.abs(K @ x - b).max() / (np.abs(K).max() * np.abs(x).max() + 1.0)\n"
        "print('RESULT', f.inertia == (n1, m, 0), res)\n" % (root, dim))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, GBOPT_LDLT_TIMING="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")][-1].split()
    assert line[1] == "True" and float(line[2]) <= 1e-10
    used = "panel" if "bkp_factor_kernel" in r.stderr else "cpanel" if "cpanel nb" in r.stderr else "grid"
    assert used == kernel, r.stderr[-1500:]

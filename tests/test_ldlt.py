"""KKT factorisation row (f3): GPU LDL^T vs the reference contract
(proj/tests/test_linalg.cpp cases restated) and the CPU oracle."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import ldlt_oracle as lo


def test_oracle_inertia_known_spectra():
    rng = np.random.default_rng(3)
    assert lo.inertia(np.eye(5)) == (5, 0, 0)
    assert lo.inertia(np.diag([2.0, -5.0])) == (1, 1, 0)
    A = lo.matrix_with_spectrum(rng, [4, 3, 2, 1, -1, -2, -3, 0])
    assert lo.inertia(A) == (4, 3, 1)
    assert lo.inertia(np.zeros((4, 4))) == (0, 0, 4)
    for n in (5, 17, 40):
        A = lo.matrix_with_spectrum(rng, rng.uniform(-3, 3, n))
        ev = np.linalg.eigvalsh(A)
        assert lo.inertia(A) == (int((ev > 0).sum()), int((ev < 0).sum()), 0)


def test_cpu_argument_checks():
    import paper_2509_22462_b200 as gb
    with pytest.raises(gb.StructuralError):
        gb.LdltFactorization(np.ones((2, 3)))
    if gb.device_count() == 0:
        # no CPU fallback: every factorisation needs the device
        with pytest.raises(gb.DeviceError):
            gb.LdltFactorization(np.eye(3))


@pytest.mark.gpu
class TestGpuLdlt:
    @pytest.fixture(autouse=True)
    def _gpu(self):
        if not has_gpu():
            pytest.skip("no GPU")

    def test_input_validation(self):
        """test_linalg.cpp:217-237: non-finite -> NumericError, asymmetric ->
        StructuralError, rhs size mismatch -> StructuralError."""
        import paper_2509_22462_b200 as gb
        with pytest.raises(gb.NumericError):
            gb.LdltFactorization(np.array([[1.0, np.nan], [np.nan, 1.0]]))
        with pytest.raises(gb.StructuralError):
            gb.LdltFactorization(np.array([[1.0, 2.0], [0.0, 1.0]]))
        f = gb.ldlt_factor(np.eye(3))
        with pytest.raises(gb.StructuralError):
            f.solve(np.ones(4))

    def test_known_inertias(self):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(3)
        assert gb.ldlt_factor(np.eye(6)).inertia == (6, 0, 0)                    # test_linalg.cpp:42
        assert gb.ldlt_factor(np.diag([2.0, -5.0])).inertia == (1, 1, 0)         # :47
        assert gb.ldlt_factor(np.array([[3.0]])).inertia == (1, 0, 0)            # :55
        assert gb.ldlt_factor(np.array([[-0.5]])).inertia == (0, 1, 0)
        z = np.array([[0.0, 1.0], [1.0, 0.0]])                                   # :63 zero diagonal
        assert gb.ldlt_factor(z).inertia == (1, 1, 0)
        A = lo.matrix_with_spectrum(rng, [4, 3, 2, 1, -1, -2, -3, 0])           # :76
        assert gb.ldlt_factor(A).inertia == (4, 3, 1)
        assert gb.ldlt_factor(np.zeros((4, 4))).inertia == (0, 0, 4)             # :211

    @pytest.mark.parametrize("n", [3, 10, 64, 200, 513])
    def test_inertia_matches_oracle_and_eigenvalues(self, n):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(n)
        eigs = rng.uniform(1, 5, n) * rng.choice([-1.0, 1.0], n)
        A = lo.matrix_with_spectrum(rng, eigs)
        got = gb.ldlt_factor(A).inertia
        assert got == lo.inertia(A) == (int((eigs > 0).sum()), int((eigs < 0).sum()), 0)

    def test_rank_deficiency_counts_zeros(self):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(11)
        eigs = np.array([3.0, -2.0, 1.5, 0.0, 0.0, -1.0])
        A = lo.matrix_with_spectrum(rng, eigs)
        f = gb.ldlt_factor(A)
        assert f.inertia == (2, 2, 2)
        with pytest.raises(gb.SingularError):
            f.solve(np.ones(6))

    @pytest.mark.parametrize("keep", [True, False])
    def test_solve_round_trip(self, keep):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(5)
        A = lo.matrix_with_spectrum(rng, rng.uniform(0.5, 4, 40) * rng.choice([-1.0, 1.0], 40))
        f = gb.ldlt_factor(A, keep_input=keep)
        for _ in range(10):
            v = rng.uniform(-1, 1, 40)
            x = f.solve(A @ v)
            assert np.abs(x - v).max() <= 1e-10

    def test_ipm_like_badly_scaled_kkt(self):
        """Barrier diagonals of 1e8 beside O(1) constraint rows (the reason
        for the Ruiz equilibration, linalg.cpp:72-84): inertia (n, m, 0) and
        a small residual."""
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(8)
        n, m = 60, 20
        Hm = lo.matrix_with_spectrum(rng, rng.uniform(1, 3, n)) + np.diag(10.0 ** rng.uniform(-2, 8, n))
        Jm = rng.uniform(-1, 1, (m, n))
        K = np.block([[Hm, Jm.T], [Jm, -1e-8 * np.eye(m)]])
        f = gb.ldlt_factor(K)
        assert f.inertia == (n, m, 0) == lo.inertia(K)
        b = rng.uniform(-1, 1, n + m)
        x = f.solve(b)
        assert np.abs(K @ x - b).max() <= 1e-8 * (np.abs(K).max() * np.abs(x).max() + np.abs(b).max())

    def test_permutation_invariance(self):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(2)
        A = lo.matrix_with_spectrum(rng, [5, -4, 3, -2, 1, 0.5, -0.25])
        p = rng.permutation(7)
        assert gb.ldlt_factor(A).inertia == gb.ldlt_factor(A[np.ix_(p, p)]).inertia == (4, 3, 0)


@pytest.mark.gpu
class TestNativeBunchKaufman:
    """The native pivoting kernel (ldlt_bk.cuh): matrices that force 2x2
    pivots and 1x1 pivots with interchanges, against eigenvalues and the
    oracle, plus solves through the same factors."""

    @pytest.fixture(autouse=True)
    def _gpu(self):
        if not has_gpu():
            pytest.skip("no GPU")

    def test_zero_diagonal_forces_2x2_pivots(self):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(21)
        n = 300
        B = rng.uniform(-1, 1, (n, n))
        A = 0.5 * (B + B.T)
        np.fill_diagonal(A, 0.0)  # every first pivot test fails: 2x2 blocks or swaps
        eig = np.linalg.eigvalsh(A)
        f = gb.ldlt_factor(A)
        assert f.inertia == (int((eig > 0).sum()), int((eig < 0).sum()), 0) == lo.inertia(A)
        b = rng.uniform(-1, 1, n)
        x = f.solve(b)
        assert np.abs(A @ x - b).max() <= 1e-9 * (np.abs(A).max() * np.abs(x).max() + 1.0)

    def test_saddle_point_blocks(self):
        """[[0, J^T], [J, 0]]: all pivots are 2x2 pairings across the blocks."""
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(22)
        m = 70
        J = rng.uniform(-1, 1, (m, m)) + 3 * np.eye(m)
        K = np.block([[np.zeros((m, m)), J.T], [J, np.zeros((m, m))]])
        f = gb.ldlt_factor(K)
        assert f.inertia == (m, m, 0)
        b = rng.uniform(-1, 1, 2 * m)
        x = f.solve(b)
        assert np.abs(K @ x - b).max() <= 1e-10 * np.abs(K).max() * max(1.0, np.abs(x).max())

    @pytest.mark.parametrize("n", [1, 2, 31, 33, 1000])
    def test_block_edges_and_larger_kkt(self, n):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(100 + n)
        m = max(1, n // 4)
        H = rng.uniform(-1, 1, (n, n))
        H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 6, n))
        J = rng.uniform(-1, 1, (m, n))
        K = np.block([[H, J.T], [J, -1e-8 * np.eye(m)]])
        f = gb.ldlt_factor(K)
        assert f.inertia == lo.inertia(K)
        b = rng.uniform(-1, 1, n + m)
        x = f.solve(b)
        assert np.abs(K @ x - b).max() <= 1e-8 * (np.abs(K).max() * np.abs(x).max() + np.abs(b).max())

    def test_deterministic(self):
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(23)
        A = lo.matrix_with_spectrum(rng, rng.uniform(-2, 2, 150))
        b = rng.uniform(-1, 1, 150)
        x0 = gb.ldlt_factor(A).solve(b)
        for _ in range(3):
            assert np.array_equal(gb.ldlt_factor(A).solve(b), x0)


@pytest.mark.gpu
class TestFactorisationKernels:
    """The three native factorisation kernels on the same matrices -- blocked
    (ldlt_bkp.cuh, default for n <= 2048), one-cluster right-looking
    (ldlt_bkc.cuh) and cooperative-grid left-looking (ldlt_bk.cuh): same
    inertia as the oracle, accurate solves through each
    (GBOPT_LDLT_KERNEL forces the path)."""

    @pytest.fixture(autouse=True)
    def _gpu(self):
        if not has_gpu():
            pytest.skip("no GPU")

    @pytest.mark.parametrize("path", ["panel", "cluster", "grid"])
    @pytest.mark.parametrize("case", ["zero_diag", "saddle", "kkt", "rank_deficient", "tiny"])
    def test_paths_agree_with_oracle(self, monkeypatch, path, case):
        import paper_2509_22462_b200 as gb
        monkeypatch.setenv("GBOPT_LDLT_KERNEL", path)
        rng = np.random.default_rng(hash(case) % 1000)
        if case == "zero_diag":
            B = rng.uniform(-1, 1, (257, 257))
            A = 0.5 * (B + B.T)
            np.fill_diagonal(A, 0.0)
        elif case == "saddle":
            J = rng.uniform(-1, 1, (90, 90)) + 3 * np.eye(90)
            A = np.block([[np.zeros((90, 90)), J.T], [J, np.zeros((90, 90))]])
        elif case == "kkt":
            n, m = 600, 150
            H = rng.uniform(-1, 1, (n, n))
            H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 6, n))
            Jm = rng.uniform(-1, 1, (m, n))
            A = np.block([[H, Jm.T], [Jm, -1e-8 * np.eye(m)]])
        elif case == "rank_deficient":
            A = lo.matrix_with_spectrum(rng, np.r_[rng.uniform(1, 3, 40), -rng.uniform(1, 3, 30), np.zeros(3)])
        else:
            A = np.array([[0.0, 2.0, 1.0], [2.0, 0.0, 0.5], [1.0, 0.5, -1.0]])
        f = gb.ldlt_factor(A)
        assert f.inertia == lo.inertia(A)
        if f.inertia[2] == 0:
            b = rng.uniform(-1, 1, A.shape[0])
            x = f.solve(b)
            assert np.abs(A @ x - b).max() <= 1e-9 * (np.abs(A).max() * np.abs(x).max() + 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("nb", ["0", "1", "7", "64", "128"])
def test_grid_kernel_panel_widths(monkeypatch, nb):
    """The grid kernel's blocked mode (GBOPT_LDLT_GRID_NB; 0 = unblocked
    left-looking) at n > 2048 (its default range) on a KKT matrix whose
    zero-ish constraint block forces many interchanges and 2x2 pivots, so
    panels end on both pivot kinds: same inertia as the oracle and accurate
    solves for every width."""
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    monkeypatch.setenv("GBOPT_LDLT_KERNEL", "grid")
    monkeypatch.setenv("GBOPT_LDLT_GRID_NB", nb)
    rng = np.random.default_rng(2100)
    n, m = 1700, 450
    H = rng.uniform(-1, 1, (n, n))
    H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 3, n))
    Jm = rng.uniform(-1, 1, (m, n))
    A = np.block([[H, Jm.T], [Jm, -1e-8 * np.eye(m)]])
    f = gb.ldlt_factor(A)
    assert f.inertia == lo.inertia(A)
    b = rng.uniform(-1, 1, A.shape[0])
    x = f.solve(b)
    assert np.abs(A @ x - b).max() <= 1e-9 * (np.abs(A).max() * np.abs(x).max() + 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("solve", ["cta", "grid"])
def test_substitution_kernels_agree(monkeypatch, solve):
    """One-CTA and grid-wide substitutions (GBOPT_LDLT_SOLVE) on the same
    factors: accurate solves, 2x2 pivots included."""
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    monkeypatch.setenv("GBOPT_LDLT_SOLVE", solve)
    rng = np.random.default_rng(41)
    for n in (1, 33, 257, 700):
        B = rng.uniform(-1, 1, (n, n))
        A = 0.5 * (B + B.T)
        np.fill_diagonal(A, 0.0 if n > 1 else 2.0)
        f = gb.ldlt_factor(A)
        if f.inertia[2]:
            continue
        b = rng.uniform(-1, 1, n)
        x = f.solve(b)
        assert np.abs(A @ x - b).max() <= 1e-9 * (np.abs(A).max() * np.abs(x).max() + 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2047, 2049, 3001])
def test_default_kernel_choice_across_thresholds(n):
    """Dimensions either side of the blocked-kernel (2048) and one-CTA
    substitution (3000) limits, through the default path."""
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    rng = np.random.default_rng(n)
    m = n // 5
    H = rng.uniform(-1, 1, (n - m, n - m))
    H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 4, n - m))
    J = rng.uniform(-1, 1, (m, n - m))
    K = np.block([[H, J.T], [J, -1e-8 * np.eye(m)]])
    f = gb.ldlt_factor(K)
    ev = np.linalg.eigvalsh(K)
    assert f.inertia == (int((ev > 0).sum()), int((ev < 0).sum()), 0)
    b = rng.uniform(-1, 1, n)
    x = f.solve(b)
    assert np.abs(K @ x - b).max() <= 1e-8 * (np.abs(K).max() * np.abs(x).max() + 1.0)

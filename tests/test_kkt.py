"""KKT assembly and inertia correction: the device
assemble_kkt / inertia_correct (paper_2509_22462_b200/csrc/kkt.cu) against
the reference's own cases (proj/tests/test_ipm.cpp:313-470, restated) and the
CPU oracle (oracle/ldlt_oracle.py: assemble_kkt, inertia_correct restated
from proj/src/ipm.cpp:466-557).

Parity: the assembled matrix and right-hand side are bit-identical to the
oracle (same additions in the same order, products rounded separately).
"""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import ldlt_oracle as lo

NO_LB = -np.inf


def spd_matrix(rng, n):
    a = rng.uniform(-1, 1, (n, n))
    return a @ a.T + n * np.eye(n)


def full_rank_rows(rng, m, n):
    return rng.uniform(-1, 1, (m, n)) + np.eye(m, n) * 3.0


def dense_builder_case():
    """test_ipm.cpp:346-407: n = 6, m = 3, unbounded entries, a duplicated
    coordinate in each triplet list, mu / dw / dc non-zero."""
    rng = np.random.default_rng(321)
    n, m = 6, 3
    lower = np.array([0.0, NO_LB, -2.0, 1.0, NO_LB, -0.5])
    x = rng.uniform(2.0, 3.0, n)
    z = rng.uniform(0.1, 1.0, n)
    z[~np.isfinite(lower)] = 0.0
    lam, grad, g = rng.uniform(-1, 1, m), rng.uniform(-1, 1, n), rng.uniform(-1, 1, m)
    hr, hc = [0, 1, 2, 3, 4, 5, 3, 3], [0, 0, 2, 1, 4, 3, 1, 3]
    hv = rng.uniform(-1, 1, 8)
    jr, jc = [0, 0, 1, 2, 2, 2], [0, 3, 2, 4, 5, 4]
    jv = rng.uniform(-1, 1, 6)
    return dict(x=x, lower=lower, z=z, lam=lam, grad_f=grad, g=g, jac_rows=jr, jac_cols=jc, jac_values=jv,
                hess_rows=hr, hess_cols=hc, hess_values=hv, mu=0.037, delta_w=0.25, delta_c=1e-3)


def naive_dense(c):
    """The test's independent builder (test_ipm.cpp:375-404), numpy."""
    n, m = c["x"].size, c["g"].size
    h = np.zeros((n, n))
    for r, cc, v in zip(c["hess_rows"], c["hess_cols"], c["hess_values"]):
        h[r, cc] += v
        if r != cc:
            h[cc, r] += v
    jac = np.zeros((m, n))
    for r, cc, v in zip(c["jac_rows"], c["jac_cols"], c["jac_values"]):
        jac[r, cc] += v
    e = np.zeros((n + m, n + m))
    e[:n, :n] = h
    b = np.isfinite(c["lower"])
    e[np.arange(n)[b], np.arange(n)[b]] += c["z"][b] / (c["x"][b] - c["lower"][b])
    e[np.arange(n), np.arange(n)] += c["delta_w"]
    e[:n, n:] = jac.T
    e[n:, :n] = jac
    e[n + np.arange(m), n + np.arange(m)] = -c["delta_c"]
    rhs = np.concatenate([-c["grad_f"] - jac.T @ c["lam"], -c["g"]])
    rhs[:n][b] += c["mu"] / (c["x"][b] - c["lower"][b])
    return e, rhs


def random_case(seed, n, m, nnz_h, nnz_j, dup=True):
    rng = np.random.default_rng(seed)
    lower = np.where(rng.uniform(size=n) < 0.6, rng.uniform(-1, 0, n), NO_LB)
    x = lower + rng.uniform(0.1, 2.0, n)
    x[~np.isfinite(lower)] = rng.uniform(-1, 1, int((~np.isfinite(lower)).sum()))
    z = np.where(np.isfinite(lower), rng.uniform(0.01, 1.0, n), 0.0)
    hr = rng.integers(0, n, nnz_h)
    hc = rng.integers(0, n, nnz_h)
    jr = rng.integers(0, m, nnz_j)
    jc = rng.integers(0, n, nnz_j)
    if dup and nnz_h > 4:
        hr[-2:], hc[-2:] = hr[:2], hc[:2]            # repeated coordinates
        hr[-3], hc[-3] = hc[2], hr[2]                # the mirror of an earlier entry
    if dup and nnz_j > 2:
        jr[-1], jc[-1] = jr[0], jc[0]
    return dict(x=x, lower=lower, z=z, lam=rng.normal(size=m), grad_f=rng.normal(size=n), g=rng.normal(size=m),
                jac_rows=jr, jac_cols=jc, jac_values=rng.normal(size=nnz_j), hess_rows=hr, hess_cols=hc,
                hess_values=rng.normal(size=nnz_h), mu=0.1 * rng.uniform(), delta_w=0.0, delta_c=0.0)


def oracle_of(c):
    return lo.assemble_kkt(c["x"], c["lower"], c["z"], c["lam"], c["grad_f"], c["g"], c["jac_rows"], c["jac_cols"],
                           c["jac_values"], c["hess_rows"], c["hess_cols"], c["hess_values"], c["mu"],
                           c["delta_w"], c["delta_c"])


# ---- oracle pins (CPU) ------------------------------------------------------

def test_oracle_bounded_variable_fold():
    """test_ipm.cpp:313-326."""
    mat, rhs = lo.assemble_kkt([1.0], [0.0], [0.1], [], [0.3], [], [], [], [], [0], [0], [2.0], 0.1)
    assert mat.shape == (1, 1)
    assert mat[0, 0] == pytest.approx(2.1) and rhs[0] == pytest.approx(-0.2)


def test_oracle_one_variable_one_constraint():
    """test_ipm.cpp:328-344: exact."""
    mat, rhs = lo.assemble_kkt([0.4], [NO_LB], [0.0], [0.0], [0.0], [0.4], [0], [0], [1.0], [0], [0], [3.0], 0.1)
    assert np.array_equal(mat, np.array([[3.0, 1.0], [1.0, 0.0]]))
    assert rhs[1] == pytest.approx(-0.4)


def test_oracle_matches_independent_dense_builder():
    """test_ipm.cpp:346-407: <= 1e-14."""
    c = dense_builder_case()
    mat, rhs = oracle_of(c)
    e, r = naive_dense(c)
    assert np.abs(mat - e).max() < 1e-14 and np.abs(rhs - r).max() < 1e-14


def test_oracle_inertia_correct_cases():
    """test_ipm.cpp:409-470."""
    rng = np.random.default_rng(77)
    n, m = 5, 2
    q, a = spd_matrix(rng, n), full_rank_rows(rng, m, n)
    K = np.block([[q, a.T], [a, np.zeros((m, m))]])
    assert lo.inertia_correct(K, n, m) == (0.0, 0.0, (5, 2, 0))
    dw, dc, inert = lo.inertia_correct(-np.eye(2), 2, 0)
    assert dw == pytest.approx(10.0) and dc == 0.0 and inert == (2, 0, 0)
    h = lo.matrix_with_spectrum(rng, [2.0, 1.0, -0.5, -1.5, 0.3])
    K = np.block([[h, a.T], [a, np.zeros((m, m))]])
    dw, dc, inert = lo.inertia_correct(K, n, m)
    assert inert == (5, 2, 0)
    ev = np.linalg.eigvalsh(K + np.diag(np.r_[np.full(n, dw), np.zeros(m)]))
    assert ((ev > 0).sum(), (ev < 0).sum()) == (5, 2)


def test_cpu_pattern_checks_and_no_fallback():
    import paper_2509_22462_b200 as gb
    with pytest.raises(gb.StructuralError):
        gb.KktPattern(3, 1, [0, 3], [0, 0], [], [])       # Hessian row out of range
    with pytest.raises(gb.StructuralError):
        gb.KktPattern(3, 1, [], [], [1], [0])             # Jacobian row out of range
    if gb.device_count() == 0:
        with pytest.raises(gb.DeviceError):
            gb.KktPattern(3, 1, [0], [0], [0], [1])


# ---- device parity ------------------------------------------------------------

@pytest.mark.gpu
class TestGpuKkt:
    @pytest.fixture(autouse=True)
    def _gpu(self):
        if not has_gpu():
            pytest.skip("no GPU")

    def assemble(self, c):
        import paper_2509_22462_b200 as gb
        return gb.assemble_kkt(c["x"], c["lower"], c["z"], c["lam"], c["grad_f"], c["g"], c["jac_rows"],
                               c["jac_cols"], c["jac_values"], c["hess_rows"], c["hess_cols"], c["hess_values"],
                               c["mu"], c["delta_w"], c["delta_c"])

    def test_reference_cases_exact(self):
        import paper_2509_22462_b200 as gb
        s = gb.assemble_kkt([1.0], [0.0], [0.1], [], [0.3], [], [], [], [], [0], [0], [2.0], 0.1)
        m0, r0 = lo.assemble_kkt([1.0], [0.0], [0.1], [], [0.3], [], [], [], [], [0], [0], [2.0], 0.1)
        assert np.array_equal(s.mat, m0) and np.array_equal(s.rhs, r0)
        assert s.mat[0, 0] == pytest.approx(2.1) and s.rhs[0] == pytest.approx(-0.2)
        s = gb.assemble_kkt([0.4], [NO_LB], [0.0], [0.0], [0.0], [0.4], [0], [0], [1.0], [0], [0], [3.0], 0.1)
        assert np.array_equal(s.mat, np.array([[3.0, 1.0], [1.0, 0.0]])) and s.rhs[1] == pytest.approx(-0.4)
        c = dense_builder_case()
        s = self.assemble(c)
        mat, rhs = oracle_of(c)
        assert np.array_equal(s.mat, mat) and np.array_equal(s.rhs, rhs)
        e, r = naive_dense(c)
        assert np.abs(s.mat - e).max() < 1e-14 and np.abs(s.rhs - r).max() < 1e-14

    @pytest.mark.parametrize("seed,n,m,nnz_h,nnz_j", [(1, 1, 0, 1, 0), (2, 7, 3, 20, 9), (3, 40, 12, 300, 80),
                                                      (4, 150, 40, 3000, 600), (5, 5, 5, 0, 0)])
    def test_random_patterns_bit_exact(self, seed, n, m, nnz_h, nnz_j):
        c = random_case(seed, n, m, nnz_h, nnz_j)
        c["delta_w"], c["delta_c"] = (0.5, 1e-3) if seed % 2 else (0.0, 0.0)
        s = self.assemble(c)
        mat, rhs = oracle_of(c)
        assert np.array_equal(s.mat, mat)
        assert np.array_equal(s.rhs, rhs)

    def test_pattern_reuse_across_iterations(self):
        import paper_2509_22462_b200 as gb
        c = random_case(9, 30, 8, 200, 60)
        pat = gb.KktPattern(30, 8, c["hess_rows"], c["hess_cols"], c["jac_rows"], c["jac_cols"])
        rng = np.random.default_rng(0)
        for it in range(3):
            c["hess_values"] = rng.normal(size=200)
            c["jac_values"] = rng.normal(size=60)
            c["mu"] = 10.0 ** -it
            s = pat.assemble(c["x"], c["lower"], c["z"], c["lam"], c["grad_f"], c["g"], c["jac_values"],
                             c["hess_values"], c["mu"])
            mat, rhs = oracle_of(c)
            assert np.array_equal(s.mat, mat) and np.array_equal(s.rhs, rhs)
        with pytest.raises(gb.StructuralError):
            pat.assemble(c["x"], c["lower"], c["z"], c["lam"], c["grad_f"], c["g"], c["jac_values"][:5],
                         c["hess_values"], 0.1)

    def test_inertia_correct_reference_cases(self):
        """test_ipm.cpp:409-470 through the device path."""
        import paper_2509_22462_b200 as gb
        rng = np.random.default_rng(77)
        n, m = 5, 2
        q, a = spd_matrix(rng, n), full_rank_rows(rng, m, n)

        def system(h):
            rows, cols = np.tril_indices(n)
            jr, jc = np.nonzero(np.ones((m, n)))
            return gb.assemble_kkt(np.zeros(n), np.full(n, NO_LB), np.zeros(n), np.zeros(m), np.zeros(n),
                                   np.zeros(m), jr, jc, a[jr, jc], rows, cols, h[rows, cols], 0.0)

        cf = gb.inertia_correct(system(q))
        assert cf.delta_w == 0.0 and cf.delta_c == 0.0 and cf.fact.inertia == (5, 2, 0)
        s = gb.assemble_kkt(np.zeros(2), np.full(2, NO_LB), np.zeros(2), [], np.zeros(2), [], [], [], [],
                            [0, 1], [0, 1], [-1.0, -1.0], 0.0)
        cf = gb.inertia_correct(s)
        assert cf.delta_w == pytest.approx(10.0) and cf.fact.inertia == (2, 0, 0)
        h = lo.matrix_with_spectrum(rng, [2.0, 1.0, -0.5, -1.5, 0.3])
        s = system(h)
        cf = gb.inertia_correct(s)
        assert cf.fact.inertia == (5, 2, 0)
        dw, dc, _ = lo.inertia_correct(s.mat, n, m)
        assert (cf.delta_w, cf.delta_c) == (dw, dc)
        # the regularised matrix's eigenvalues agree
        corr = s.mat + np.diag(np.r_[np.full(n, cf.delta_w), np.zeros(m)])
        ev = np.linalg.eigvalsh(corr)
        assert ((ev > 0).sum(), (ev < 0).sum()) == (5, 2)

    def test_inertia_correct_delta_c_and_singular(self):
        import paper_2509_22462_b200 as gb
        # duplicated constraint rows: zero pivots with m > 0 -> delta_c
        n, m = 4, 2
        rng = np.random.default_rng(5)
        q = spd_matrix(rng, n)
        row = rng.uniform(-1, 1, n)
        rows, cols = np.tril_indices(n)
        jr = np.repeat([0, 1], n)
        jc = np.tile(np.arange(n), 2)
        s = gb.assemble_kkt(np.zeros(n), np.full(n, NO_LB), np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(m),
                            jr, jc, np.r_[row, row], rows, cols, q[rows, cols], 0.0)
        cf = gb.inertia_correct(s)
        dw, dc, inert = lo.inertia_correct(s.mat, n, m)
        assert cf.fact.inertia == inert == (n, m, 0)
        assert cf.delta_c > 0.0 and (cf.delta_w, cf.delta_c) == (dw, dc)
        # escalation past delta_max -> SingularError
        s = gb.assemble_kkt(np.zeros(2), np.full(2, NO_LB), np.zeros(2), [], np.zeros(2), [], [], [], [],
                            [0, 1], [0, 1], [-1e3, -1e3], 0.0)
        with pytest.raises(gb.SingularError):
            gb.inertia_correct(s, gb.IpmOptions(delta_max=100.0))

    def test_device_rhs_solve_matches_host_solve(self):
        import paper_2509_22462_b200 as gb
        c = random_case(11, 60, 15, 500, 120)
        rows, cols = np.tril_indices(60)
        rng = np.random.default_rng(2)
        h = spd_matrix(rng, 60)
        c.update(hess_rows=rows, hess_cols=cols, hess_values=h[rows, cols])
        s = self.assemble(c)
        cf = gb.inertia_correct(s)
        x_dev = s.solve(cf.fact)
        x_host = cf.fact.solve(s.rhs)
        assert np.array_equal(x_dev, x_host)
        mat = s.mat
        assert np.abs(mat @ x_dev - s.rhs).max() <= 1e-9 * (np.abs(mat).max() * np.abs(x_dev).max() + 1.0)

    def test_reduced_space_newton_system(self):
        """The IPM's Newton system for a reduced-space NN block: the
        callbacks' triplets (reduced_space.py, formulations.cpp:267-349) with
        an objective Hessian added on the diagonal, assembled and factored on
        the device, solved through the device rhs."""
        import paper_2509_22462_b200 as gb
        from paper_2509_22462_b200.reduced_space import ReducedSpaceBlock
        net = gb.random_net([12, 16, 16, 3], "tanh", "linear", 4).bind_device(0)
        blk = ReducedSpaceBlock(net)
        n, m = blk.n + blk.m, blk.m
        rng = np.random.default_rng(3)
        xb = np.concatenate([rng.uniform(0, 1, blk.n), rng.normal(size=blk.m)])
        lam = rng.normal(size=m)
        jr, jc = blk.jac_pattern()
        hr, hc = blk.hess_pattern()
        # objective: 0.5 |xb|^2 -> identity Hessian on every variable
        hr2 = np.r_[hr, np.arange(n)]
        hc2 = np.r_[hc, np.arange(n)]
        hv = np.r_[blk.lag_hessian(xb, lam), np.ones(n)]
        lower = np.r_[np.zeros(blk.n), np.full(blk.m, NO_LB)]
        x = xb + np.r_[np.full(blk.n, 0.5), np.zeros(blk.m)]
        z = np.r_[np.full(blk.n, 0.1), np.zeros(blk.m)]
        c = dict(x=x, lower=lower, z=z, lam=lam, grad_f=xb, g=blk.residual(xb), jac_rows=jr, jac_cols=jc,
                 jac_values=blk.jacobian(xb), hess_rows=hr2, hess_cols=hc2, hess_values=hv, mu=0.01,
                 delta_w=0.0, delta_c=0.0)
        pat = gb.KktPattern(n, m, hr2, hc2, jr, jc)
        s = pat.assemble(x, lower, z, lam, xb, c["g"], c["jac_values"], hv, 0.01)
        mat, rhs = oracle_of(c)
        assert np.array_equal(s.mat, mat) and np.array_equal(s.rhs, rhs)
        cf = gb.inertia_correct(s)
        dw, dc, inert = lo.inertia_correct(mat, n, m)
        assert cf.fact.inertia == inert == (n, m, 0) and (cf.delta_w, cf.delta_c) == (dw, dc)
        sol = s.solve(cf.fact)
        corr = mat + np.diag(np.r_[np.full(n, cf.delta_w), np.full(m, -cf.delta_c)])
        assert np.abs(corr @ sol - rhs).max() <= 1e-10 * (np.abs(corr).max() * np.abs(sol).max() + 1.0)


@pytest.mark.gpu
def test_kkt_without_constraints_and_large_system():
    """m = 0 (no constraint block, delta_c never used) and a dimension past
    the blocked factorisation's limit (grid kernel inside inertia_correct)."""
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    rng = np.random.default_rng(12)
    n = 40
    q = spd_matrix(rng, n) - 2.5 * n * np.eye(n)   # indefinite: needs delta_w
    rows, cols = np.tril_indices(n)
    s = gb.assemble_kkt(np.zeros(n), np.full(n, NO_LB), np.zeros(n), [], rng.normal(size=n), [], [], [], [],
                        rows, cols, q[rows, cols], 0.0)
    cf = gb.inertia_correct(s)
    dw, dc, inert = lo.inertia_correct(s.mat, n, 0)
    assert cf.fact.inertia == inert == (n, 0, 0) and (cf.delta_w, cf.delta_c) == (dw, dc) and cf.delta_w > 0
    n, m = 2000, 400
    c = random_case(13, n, m, 6000, 3000)
    rows, cols = np.tril_indices(n)
    h = np.diag(rng.uniform(1, 2, n))
    c.update(hess_rows=np.r_[c["hess_rows"], np.arange(n)], hess_cols=np.r_[c["hess_cols"], np.arange(n)],
             hess_values=np.r_[c["hess_values"], 50.0 * np.ones(n)])
    pat = gb.KktPattern(n, m, c["hess_rows"], c["hess_cols"], c["jac_rows"], c["jac_cols"])
    sys_ = pat.assemble(c["x"], c["lower"], c["z"], c["lam"], c["grad_f"], c["g"], c["jac_values"], c["hess_values"],
                        c["mu"])
    mat, rhs = oracle_of(c)
    assert np.array_equal(sys_.mat, mat) and np.array_equal(sys_.rhs, rhs)
    cf = gb.inertia_correct(sys_)
    assert cf.fact.inertia == (n, m, 0)
    sol = sys_.solve(cf.fact)
    corr = mat + np.diag(np.r_[np.full(n, cf.delta_w), np.full(m, -cf.delta_c)])
    assert np.abs(corr @ sol - rhs).max() <= 1e-8 * (np.abs(corr).max() * np.abs(sol).max() + 1.0)

"""Small f3 workload for compute-sanitizer: KKT assembly, inertia
correction and solves through each factorisation kernel (blocked, cluster-panel,
cluster, grid) and both substitutions.  python tools/sanitize_f3.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402

rng = np.random.default_rng(0)
n, m = 90, 20
H = rng.uniform(-1, 1, (n, n))
H = 0.5 * (H + H.T)
J = rng.uniform(-1, 1, (m, n))
rows, cols = np.tril_indices(n)
jr, jc = np.nonzero(np.ones((m, n)))
for kern in ("panel", "cpanel", "cluster", "grid"):
    os.environ["GBOPT_LDLT_KERNEL"] = kern
    for sv in ("cta", "grid"):
        os.environ["GBOPT_LDLT_SOLVE"] = sv
        s = gb.assemble_kkt(np.ones(n), np.zeros(n), np.full(n, 0.1), rng.normal(size=m), rng.normal(size=n),
                            rng.normal(size=m), jr, jc, J[jr, jc], rows, cols, H[rows, cols], 0.01)
        cf = gb.inertia_correct(s)
        x = s.solve(cf.fact)
        K = s.mat + np.diag(np.r_[np.full(n, cf.delta_w), np.full(m, -cf.delta_c)])
        print(kern, sv, cf.fact.inertia, cf.delta_w, float(np.abs(K @ x - s.rhs).max()))

# the cluster-panel kernel over several panels (displaced rows carried across
# compactions, 2 rows per thread at the tail of the slice)
os.environ["GBOPT_LDLT_KERNEL"] = "cpanel"
n1, m1 = 150, 60
H1 = rng.uniform(-1, 1, (n1, n1))
K1 = np.block([[0.5 * (H1 + H1.T), rng.uniform(-1, 1, (n1, m1))], [np.zeros((m1, n1)), np.zeros((m1, m1))]])
K1[n1:, :n1] = K1[:n1, n1:].T
f1 = gb.ldlt_factor(K1)
b1 = rng.uniform(-1, 1, n1 + m1)
print("cpanel multi-panel", f1.inertia, float(np.abs(K1 @ f1.solve(b1) - b1).max()))

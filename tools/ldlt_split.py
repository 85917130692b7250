import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import paper_2509_22462_b200 as gb
def kkt(n, m, seed):
    rng = np.random.default_rng(seed)
    H = rng.uniform(-1, 1, (n, n)); H = 0.5 * (H + H.T) + np.diag(10.0 ** rng.uniform(-2, 6, n))
    J = rng.uniform(-1, 1, (m, n))
    return np.block([[H, J.T], [J, -1e-8 * np.eye(m)]]), rng.uniform(-1, 1, n + m)
if __name__ == "__main__":
  for n in [int(v) for v in sys.argv[1:]] or (784, 2000, 4000, 8000):
      K, b = kkt(n, n // 8, n)
      f = gb.ldlt_factor(K); f.solve(b)
      t0 = time.perf_counter(); f = gb.ldlt_factor(K); t1 = time.perf_counter(); x = f.solve(b); t2 = time.perf_counter()
      print(K.shape[0], "factor %.2f ms solve %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3), "resid", np.abs(K @ x - b).max())

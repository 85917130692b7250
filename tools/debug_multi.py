import faulthandler, sys, os
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_22462_b200 import configs
batch, S = int(sys.argv[1]), int(sys.argv[2])
wl = configs.make("c4", batch=batch)
net = wl.net.bind_device(0)
print("single", flush=True)
Y0, J0, H0 = net.oracle_batched(wl.X, wl.Lam)
print("multi", flush=True)
Y, J, H = net.oracle_batched_multi([0] * S, wl.X, wl.Lam)
print("multi done", flush=True)
for r in range(S):
    c = batch // S + (1 if r < batch % S else 0)
    s = r * (batch // S) + min(r, batch % S)
    y1, j1, h1 = net.oracle_batched(wl.X[s:s + c], wl.Lam[s:s + c])
    print(r, s, c, np.array_equal(Y[s:s+c], y1), np.array_equal(J[s:s+c], j1), np.array_equal(H[s:s+c], h1),
          np.abs(H[s:s+c] - h1).max(), np.abs(H[s:s+c]-H0[s:s+c]).max(), flush=True)

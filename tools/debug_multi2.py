import faulthandler, sys, os
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_22462_b200 import configs
batch, S, graphs, warm = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "1", sys.argv[4] == "1"
wl = configs.make("c4", batch=batch)
net = wl.net.bind_device(0)
net.set_graphs(graphs)
if warm:
    for r in range(S):
        c = batch // S + (1 if r < batch % S else 0)
        net.oracle_batched(wl.X[:c], wl.Lam[:c])
try:
    Y, J, H = net.oracle_batched_multi([0] * S, wl.X, wl.Lam)
    print("ok", batch, S, graphs, warm)
except Exception as e:
    print("FAIL", batch, S, graphs, warm, e)

"""GBNN load + device upload of the c2 net: save once, then time
load_weights (file -> host Net) and bind_device (host -> HBM, kernel layout)
separately, and the first evaluation.  python tools/load_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_22462_b200 as gb  # noqa: E402
from paper_2509_22462_b200 import configs  # noqa: E402

wl = configs.make("c2", batch=1)
path = "/tmp/c2_probe.gbnn"
t0 = time.perf_counter()
gb.save_weights(wl.net, path)
t1 = time.perf_counter()
print(f"save {t1 - t0:.3f} s  ({os.path.getsize(path) / 1e6:.1f} MB)")
for rep in range(2):
    t0 = time.perf_counter()
    net = gb.load_weights(path)
    t1 = time.perf_counter()
    net.bind_device(0)
    t2 = time.perf_counter()
    y = net.forward(wl.X[0])
    t3 = time.perf_counter()
    print(f"load {t1 - t0:.3f} s  bind {t2 - t1:.3f} s  first forward {t3 - t2:.3f} s")
    del net
os.remove(path)

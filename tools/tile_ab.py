import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2509_22462_b200 as gb
B = 32
net = gb.random_net([784, 5120, 5120, 10], "linear", "linear", 3)
rng = np.random.default_rng(0)
X = rng.uniform(0, 1, (B, 784)); L = rng.normal(0, 1, (B, 10))
dev = torch.device("cuda", 0)
Xd = torch.from_numpy(X).to(dev); Ld = torch.from_numpy(L).to(dev)
net.bind_device(0)
net.set_schedule("layered"); net.oracle_batched(X, L)
for _ in range(2):
    recs = gb.gbopt.profile_launches(net, B, Xd.data_ptr(), Ld.data_ptr())
g = [r for r in recs if r[0] == "nt_mma.gemm"]
tiles = B * 7 * 40
print("layered gemm launches", [round(r[1], 3) for r in g], "tiles", tiles, "waves", tiles / 148, "us/tile(packed)", g[0][1] * 1e3 * 148 / tiles)
net.set_schedule("dataflow"); net.oracle_batched(X, L)
for _ in range(2):
    tr = gb.gbopt.dataflow_trace(net, B, Xd.data_ptr(), Ld.data_ptr())
k = tr[:, 0].astype(int)
d = tr[:, 11] - tr[:, 10]
print("df gemm us/tile mean", d[k == 2].mean(), "min", d[k == 2].min(), "span ms", tr[:, 11].max() / 1e3)
gaps = []
for sm in np.unique(tr[:, 7]):
    s = np.where((tr[:, 7] == sm) & (k == 2))[0]
    s = s[np.argsort(tr[s, 10])]
    gaps.extend(tr[s[1:], 10] - tr[s[:-1], 11])
print("df gap between consecutive gemm tiles on an SM: mean", np.mean(gaps), "us")
# clocks while each schedule runs back to back for ~2 s
import subprocess, threading, time
def sample(out, stop):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active", "--format=csv,noheader"], capture_output=True, text=True)
        out.append(r.stdout.strip()); time.sleep(0.2)
for sched in ("layered", "dataflow"):
    net.set_schedule(sched); net.oracle_batched(X, L)
    out, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(out, stop)); th.start()
    Y = torch.empty(B, 10, dtype=torch.float64, device=dev); J = torch.empty(B, 10, 784, dtype=torch.float64, device=dev); H = torch.empty(B, 784, 784, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    t0 = time.time()
    while time.time() - t0 < 3:
        for _ in range(10):
            net.oracle_batched_device(B, Xd.data_ptr(), Ld.data_ptr(), Y.data_ptr(), J.data_ptr(), H.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
    stop.set(); th.join()
    print(sched, out[len(out)//3:len(out)//3+6])

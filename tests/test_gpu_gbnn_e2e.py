"""f2 end to end: the BASELINE c2 network (softplus, GBNN code
4, 871.6 MB) written as a GBNN v1 file, loaded by the product's reader
(nn_io.cpp:144-221 restated, parallel pread), uploaded to HBM, evaluated on
the device -- and checked against the CPU oracle reading THE SAME BYTES with
its own independent GBNN reader (oracle/gbopt_oracle.py load_weights_bytes,
which accepts code 4 like the product).  The load and upload times are
printed (profiles/r02_gbnn_load.txt)."""
import os
import time

import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as orc

pytestmark = pytest.mark.gpu


def test_c2_gbnn_file_to_device_parity(tmp_path):
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs
    wl = configs.make("c2", batch=1)
    path = str(tmp_path / "c2.gbnn")
    gb.save_weights(wl.net, path)
    size = os.path.getsize(path)
    assert size == 12 + sum(9 + 8 * (r * c + r) for r, c in
                            [(wl.net.layer(l)[0].shape) for l in range(wl.net.layer_count)])
    t0 = time.perf_counter()
    net = gb.load_weights(path)
    t1 = time.perf_counter()
    net.bind_device(0)
    t2 = time.perf_counter()
    x, lam = wl.X[0], wl.Lam[0]
    y, j, h = net.oracle(x, lam)
    t3 = time.perf_counter()
    assert all(net.layer(l)[2] == gb.SOFTPLUS for l in range(net.layer_count - 1))
    # the oracle parses the same bytes with its own reader
    with open(path, "rb") as f:
        onet = orc.load_weights_bytes(f.read())
    for l in range(net.layer_count):
        w, b, a = net.layer(l)
        assert np.array_equal(w, onet.layers[l].weight) and np.array_equal(b, onet.layers[l].bias)
        assert a == onet.layers[l].activation
    assert orc.rel_err(y, onet.forward(x)) <= 1e-10
    assert orc.rel_err(j, onet.jacobian(x)) <= 1e-10
    assert orc.rel_err(h, onet.lagrangian_hessian(x, lam)) <= 1e-10
    print(f"\nGBNN c2 {size / 1e6:.1f} MB: load_weights {t1 - t0:.3f} s ({size / (t1 - t0) / 1e9:.2f} GB/s), "
          f"bind_device (upload, kernel layout) {t2 - t1:.3f} s ({size / (t2 - t1) / 1e9:.2f} GB/s), "
          f"first oracle call {t3 - t2:.3f} s")

"""forward() (the line-search residual, nn.cpp:113-125) and forward_trace()
(nn.cpp:127-146) through both single-point paths: the default per-layer GEMV
graph and the opt-in persistent launch (csrc/fwd_stream.cuh,
GBOPT_FWD_STREAM=1: one cooperative launch streaming every layer's weights
with 1-D TMA bulk copies).  Checked against the CPU oracle on nets that exercise each
chunk geometry (several rows per chunk, one row per chunk, rows split into
segments wider than a chunk, fewer rows than SMs, softmax output), against
the per-layer GEMV path (GBOPT_FWD_STREAM=0, separate process), and for
bitwise determinism."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import has_gpu
from oracle import gbopt_oracle as orc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

NETS = [
    ([784, 5120, 5120, 10], "softplus", "linear", 1),   # 1 row per chunk (40 KB rows)
    ([100, 300, 200, 7], "tanh", "softmax", 2),         # many rows per chunk, softmax output
    ([37, 6000, 9], "sigmoid", "tanh", 3),               # 6000-wide rows: 2 segments per row
    ([5, 3], "tanh", "linear", 4),                       # fewer rows than SMs
    ([64] + [256] * 30 + [4], "sigmoid", "linear", 5),   # deep chain: 31 inter-layer barriers
]


def _net(widths, hid, fin, seed):
    import paper_2509_22462_b200 as gb
    return gb.random_net(widths, hid, fin, seed).bind_device(0)


@pytest.mark.parametrize("mode", ["1", "0"])
@pytest.mark.parametrize("widths,hid,fin,seed", NETS)
def test_forward_stream_matches_oracle(monkeypatch, widths, hid, fin, seed, mode):
    if not has_gpu():
        pytest.skip("no GPU")
    monkeypatch.setenv("GBOPT_FWD_STREAM", mode)  # read when the handle binds
    net = _net(widths, hid, fin, seed)
    on = orc.NeuralNet([orc.Layer(*net.layer(l)) for l in range(net.layer_count)])
    rng = np.random.default_rng(seed)
    for _ in range(2):
        x = rng.uniform(-1, 1, widths[0])
        y = net.forward(x)
        assert orc.rel_err(y, on.forward(x)) <= 1e-13
        z_g, y_g = net.forward_trace(x)
        z_o, y_o = on.forward_trace(x)
        for l in range(len(z_o)):
            assert orc.rel_err(z_g[l], z_o[l]) <= 1e-13 and orc.rel_err(y_g[l], y_o[l]) <= 1e-13
        assert np.array_equal(y_g[-1], y)
        assert np.array_equal(net.forward(x), y)  # bitwise repeatable


_SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2509_22462_b200 as gb
net = gb.random_net({widths!r}, {hid!r}, {fin!r}, {seed}).bind_device(0)
x = np.random.default_rng(9).uniform(-1, 1, {n})
print(json.dumps(net.forward(x).tolist()))
"""


@pytest.mark.parametrize("widths,hid,fin,seed", NETS[:3])
def test_forward_stream_agrees_with_per_layer_path(widths, hid, fin, seed):
    if not has_gpu():
        pytest.skip("no GPU")
    outs = []
    for mode in ("1", "0"):  # opt-in persistent launch vs the default per-layer graph
        code = _SCRIPT.format(root=ROOT, widths=widths, hid=hid, fin=fin, seed=seed, n=widths[0])
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, GBOPT_FWD_STREAM=mode))
        assert r.returncode == 0, r.stderr
        outs.append(np.array(json.loads(r.stdout.strip().splitlines()[-1])))
    assert orc.rel_err(outs[0], outs[1]) <= 1e-14

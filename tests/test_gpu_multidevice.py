"""Multi-device evaluation inside one process (gbopt_net_oracle_batched_multi
and _multi_gather, csrc/multi.cpp): replicas of one handle's weights, one
host thread per slot, contiguous shards, no reduction.

The pool gives one GPU per call, so the slots are replicas on device 0
(independent workspaces and streams).  GBOPT_MULTI_STAGE=1 sends every slot
but the first through the remote path (staging buffers + cudaMemcpyPeerAsync
pull of x / lambda and push of the results), so the gather code runs here
exactly as it would between two GPUs.  Each shard must be bit-identical to
evaluating it alone on one device.
"""
import numpy as np
import pytest

from conftest import has_gpu

if has_gpu():
    import paper_2509_22462_b200 as gb
    from paper_2509_22462_b200 import configs


def shards(B, S):
    out = []
    for r in range(S):
        c = B // S + (1 if r < B % S else 0)
        s = r * (B // S) + min(r, B % S)
        out.append((s, c))
    return out


def test_multi_argument_checks():
    import paper_2509_22462_b200 as g
    net = g.random_net([4, 5, 2], "tanh", "linear", 1)
    with pytest.raises(g.ArgumentError):
        net.oracle_batched_multi([], np.zeros((2, 4)), np.zeros((2, 2)))
    with pytest.raises(g.ArgumentError):
        net.oracle_batched_multi([0], np.zeros((2, 3)), np.zeros((2, 2)))
    if g.device_count() == 0:
        with pytest.raises(g.DeviceError):
            net.oracle_batched_multi([0, 0], np.zeros((2, 4)), np.zeros((2, 2)))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,batch,S", [("c4", 64, 2), ("c4", 67, 3), ("c5", 4, 2)])
def test_multi_host_shards_bitwise(cfg, batch, S):
    if not has_gpu():
        pytest.skip("no GPU")
    wl = configs.make(cfg, batch=batch)
    net = wl.net.bind_device(0)
    Y, J, H = net.oracle_batched_multi([0] * S, wl.X, wl.Lam)
    for s, c in shards(batch, S):
        y1, j1, h1 = net.oracle_batched(wl.X[s:s + c], wl.Lam[s:s + c])
        assert np.array_equal(Y[s:s + c], y1) and np.array_equal(J[s:s + c], j1) and np.array_equal(H[s:s + c], h1)


@pytest.mark.gpu
@pytest.mark.parametrize("stage", ["0", "1"])
def test_multi_gather_on_device0(monkeypatch, stage):
    if not has_gpu():
        pytest.skip("no GPU")
    import torch
    monkeypatch.setenv("GBOPT_MULTI_STAGE", stage)
    wl = configs.make("c4", batch=96)
    net = wl.net.bind_device(0)
    B, n, m = 96, net.input_dim, net.output_dim
    dX = torch.from_numpy(wl.X).cuda()
    dL = torch.from_numpy(wl.Lam).cuda()
    dY = torch.full((B, m), np.nan, dtype=torch.float64, device="cuda")
    dJ = torch.full((B, m, n), np.nan, dtype=torch.float64, device="cuda")
    dH = torch.full((B, n, n), np.nan, dtype=torch.float64, device="cuda")
    net.oracle_batched_multi_gather([0, 0, 0], B, dX.data_ptr(), dL.data_ptr(), dY.data_ptr(), dJ.data_ptr(),
                                    dH.data_ptr())
    Y, J, H = net.oracle_batched_multi([0, 0, 0], wl.X, wl.Lam)
    assert np.array_equal(dY.cpu().numpy(), Y)
    assert np.array_equal(dJ.cpu().numpy(), J)
    assert np.array_equal(dH.cpu().numpy(), H)

"""Distinct handles may run on distinct host threads at once (gbopt.h
convention, nn.hpp:38-39): two handles of one net evaluated concurrently on
one GPU must give bit-identical results to a single-threaded evaluation --
the full oracle (tangent GEMMs, SYRKs, forward, adjoint) and the
reverse-mode Jacobian.  (This is what exposed the DMMA skinny adjoint's
wrong-partials race, now opt-in: csrc/kernels.cuh, profiles/r02_notes.md.)"""
import threading

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu


def _run_two(make_net, call, reps):
    want = call(make_net())
    nets = [make_net(), make_net()]
    bad = []

    def work(t):
        for r in range(reps):
            got = call(nets[t])
            for a, b in zip(got if isinstance(got, tuple) else (got,), want if isinstance(want, tuple) else (want,)):
                if not np.array_equal(a, b):
                    bad.append((t, r))
                    return

    ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return bad


@pytest.mark.parametrize("widths,hid,fin,B", [
    ([256, 1024, 1024, 1024, 10], "sigmoid", "linear", 6),
    ([108, 512, 512, 1], "tanh", "sigmoid", 300),
])
def test_two_handles_concurrent_oracle_bitwise(widths, hid, fin, B):
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    rng = np.random.default_rng(B)
    X = rng.uniform(-1, 1, (B, widths[0]))
    L = rng.normal(size=(B, widths[-1]))
    bad = _run_two(lambda: gb.random_net(widths, hid, fin, 7).bind_device(0), lambda n: n.oracle_batched(X, L), 15)
    assert not bad, bad


def test_two_handles_concurrent_reverse_jacobian_bitwise():
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2509_22462_b200 as gb
    widths = [784, 5120, 5120, 5120, 10]  # c2-wide layers: 2 DMMA-adjoint CTAs per SM
    x = np.random.default_rng(3).uniform(0, 1, widths[0])
    bad = _run_two(lambda: gb.random_net(widths, "tanh", "linear", 5).bind_device(0), lambda n: n.jacobian(x), 150)
    assert not bad, bad

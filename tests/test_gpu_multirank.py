"""The N > 1 path on the device: `bench.py --gpus 2` launches two ranks
itself (no torchrun on the command line), each rank runs the device oracle
on its shard, packs, and gathers to rank 0, which checks the gathered
(y, J, H) bit for bit against the same shards evaluated by one process.

The pool gives one GPU per call, so both ranks share device 0 and the
gather runs over gloo (NCCL refuses two ranks on one GPU); this is a
correctness run of the data path, not a performance number (the JSON line
says so).  On an 8-GPU box the same code runs over NCCL.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["c2", "c4"])
def test_two_ranks_gather_bitwise(config):
    if not has_gpu():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                        "--config", config, "--steps", "2", "--warmup", "1", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2
    mr = line["multi_rank"]
    assert mr["backend"] == "gloo" and mr["bitwise_equal_to_single_process_shards"] is True
    assert mr["gathered_points"] == (2 if config == "c2" else 4096)
    assert line["parity"]["pass"] is True
    assert line["e2e"]["value"] > 0
    if config == "c2":
        recs = {s["config"]: s for s in line["sharded"]}
        assert recs["c3"]["points_total"] == 64 and recs["c3"]["points_per_gpu_max"] == 32
        assert recs["c4"]["points_total"] == 4096 and recs["c4"]["points_per_gpu_max"] == 2048

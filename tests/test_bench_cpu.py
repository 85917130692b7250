"""bench.py's CPU reference arm (the driver runs `bench.py --impl reference`)
emits the contract's JSON line; runs here on the small config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@needs_ref
def test_reference_arm_json_line_and_no_product_library():
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '2', "
            "'--warmup', '1'];\ntry:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('PRODUCT_SO_LOADED' if 'libgbopt_b200' in maps else 'PRODUCT_SO_ABSENT')\n"
            "print('REF_SO_LOADED' if 'libgbopt_ref' in maps else 'REF_SO_ABSENT')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    out = r.stdout.strip().splitlines()
    assert out[-2] == "PRODUCT_SO_ABSENT" and out[-1] == "REF_SO_LOADED", out[-2:]
    line = json.loads(out[-3])
    for key in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    import bench
    assert line["config"] == bench.config_dict("c1", 1)


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--gpus", "2", "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_bench_flops_and_config_tables_match_the_generators(name):
    import bench
    from paper_2509_22462_b200 import configs
    assert bench.flops_per_eval(name) == configs.flops(name)
    assert bench.WIDTHS[name] == configs.CONFIGS[name]["widths"] == ref.CONFIGS[name]["widths"]
    assert bench.TOTAL_POINTS[name] == configs.CONFIGS[name]["batch"] == ref.CONFIGS[name]["batch"]
    assert (name in bench.SOFTPLUS_CONFIGS) == (ref.CONFIGS[name]["hidden"] == ref.SOFTPLUS)


def test_gpus_n_without_launcher_spawns_ranks(tmp_path):
    """`bench.py --gpus 2` outside torchrun starts two ranks (here each rank
    fails fast for lack of a GPU, which proves both were launched)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "1", "--config", "c1"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode != 0
    assert "torch.distributed.run" in r.stderr or "ChildFailedError" in r.stderr or "rank" in r.stderr.lower()

"""bench.py's launcher on CPU: `--gpus 2` without a torchrun environment
starts two ranks itself; with no CUDA device they join a gloo group and run
the exchange plumbing (dry run), and rank 0 reports both ranks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(300)
def test_bench_gpus_2_launches_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--n", "3001",
                          "--dry-run"], capture_output=True, text=True, timeout=280, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["comm"]["ranks_reporting"] == 2 and d["comm"]["exchange_ok"]
    assert d["comm"]["padded_elements"] % 8 == 0 and d["comm"]["padded_elements"] >= d["comm"]["packed_elements"]
    assert d["config"]["name"] == "cfg4"


def test_bench_presets_follow_baseline_configs():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2510_12174_b200 import scenes
    for name, p in bench.PRESETS.items():
        c = scenes.CONFIGS[name]
        assert (p["n"], p["width"], p["height"], p["focal"], p["classes"]) == \
            (c["n"], c["width"], c["height"], c["f"], c["C"])
        assert p["mode"] == ("fwd" if c["passes"] == "fwd" else "fwdbwd")
    a = bench.parse(["--config", "cfg5", "--n", "10"])
    assert a.n == 10 and a.width == 1920 and a.mode == "fwd"

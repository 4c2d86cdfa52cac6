"""GPU check of bench.py's own arm at a small scale: the single-GPU line and the
multi-rank path at world 1 (torch.distributed NCCL group + the library's NCCL
communicator + shard load + per-iteration exchange, `--dist`) both print one JSON
line with the contract's keys, and the values the two report agree."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "per_algo")


def run_bench(*extra):
    env = dict(os.environ, MASTER_PORT=str(29600 + os.getpid() % 1000))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--shift", "8",
                          "--steps", "1", "--warmup", "3", "--e2e-steps", "1", "--no-extras", "--no-cpu-baseline",
                          *extra], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("dist", [False, True], ids=["single", "nccl_world1"])
def test_bench_line(dist):
    line = run_bench(*(["--dist"] if dist else []))
    for k in KEYS:
        assert k in line, k
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["per_algo"]["sssp"]["iterations"] > 0 and line["per_algo"]["pr"]["iterations"] > 0
    if dist:
        assert "NCCL" in line["config"]["parallelism"]
        assert "exchange" in line["per_algo"]["pr"]
        assert "shard" in line["e2e"]["includes"]

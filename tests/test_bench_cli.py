"""bench.py's multi-rank plumbing on CPU: `--gpus N` without
torchrun re-launches itself under torch.distributed.run with N ranks; each
rank owns a contiguous batch shard (paper_1904_08368_b200.shard) and the
shards cover the global batch in order.  --dry-run stops before any GPU work
(gloo world, all_gather of the plan to rank 0)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run"] + list(args),
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_single_gpu_default_line():
    d = _run()
    assert d["n_gpus"] == 1 and d["ranks"] == [{"rank": 0, "world": 1, "shard": [0, 256]}]
    assert d["config"]["workload"] == "resnet18_int8_b256"


@pytest.mark.parametrize("gpus,gb", [(2, 0), (2, 4096), (3, 4096)])
def test_gpus_n_spawns_n_ranks(gpus, gb):
    d = _run("--gpus", str(gpus), *(["--global-batch", str(gb)] if gb else []))
    assert d["n_gpus"] == gpus
    assert sorted(r["rank"] for r in d["ranks"]) == list(range(gpus))
    shards = [r["shard"] for r in sorted(d["ranks"], key=lambda r: r["rank"])]
    total = gb or 256 * gpus
    assert shards[0][0] == 0 and shards[-1][1] == total
    assert all(shards[i][1] == shards[i + 1][0] for i in range(gpus - 1))
    assert d["config"]["workload"] == "resnet18_int8_b%d" % total


def test_model_flag_labels_the_workload():
    d = _run("--model", "mobilenet_v1")
    assert d["config"]["workload"] == "mobilenet_v1_int8_b256"
    assert "MobileNet" in d["config"]["model"]
    d = _run("--model", "vgg16_b256")
    assert d["config"]["workload"] == "vgg16_b256_bf16_b256"

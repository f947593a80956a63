"""Multi-GPU path on CPU: contiguous batch shards, one per
rank, no collective on the data path.  World-size-2 gloo processes each run
their shard through the CPU oracle and the gathered shards must equal the
unsharded reference output bit for bit (per-sample independence), exactly
what bench.py --gpus N relies on."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1904_08368_b200.shard import shard_range, shard_sizes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("total,world", [(4096, 8), (256, 3), (5, 2), (1, 4), (0, 2)])
def test_shard_range_partitions(total, world):
    seen = []
    for r in range(world):
        a, b = shard_range(total, r, world)
        seen += list(range(a, b))
    assert seen == list(range(total))
    s = shard_sizes(total, world)
    assert max(s) - min(s) <= 1 and sum(s) == total


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1904_08368_b200 as mrb
        from paper_1904_08368_b200 import modelzoo
        from oracle import port as oport
        oport.set_threads(2)
        text, meta, src = mrb.load_model("resnet18_tiny", "int8")
        w = modelzoo.make_weights(src, seed=meta["weights_seed"])
        x = modelzoo.make_inputs(src, 4, seed=0)  # the global batch of the golden fixture
        a, b = shard_range(4, rank, world)
        # each rank compiles its module at its own shard size (as bench.py does)
        assert mrb.lower(text, batch=b - a)["result_shape"] == [b - a, 10]
        y = oport.run_weights(text, x[a:b], [w[p.name] for p in src.params if p.kind != "input"])
        parts = [None] * world
        dist.all_gather_object(parts, (a, y))  # result collection only, after the data path
        if rank == 0:
            q.put(np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])]))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_equal_unsharded_golden():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    y = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gold = np.load(os.path.join(ROOT, "tests", "golden", "resnet18_tiny_b4.npz"))["int8"]
    assert np.array_equal(y.view(np.uint32), gold.view(np.uint32))

"""Multi-process host logic of the batched configuration (configs[4]) on CPU: world size 2
over gloo (127.0.0.1), as the 8-GPU runs use it over NCCL (-m "not gpu")."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2510_02126_b200 import batch  # noqa: E402


def test_shard_partitions_exactly():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            parts = [batch.shard(n, r, world) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))                       # disjoint, complete, ordered
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_stratified_sample_keeps_every_kappa_group():
    idx = batch.stratified(256, 4, 2)
    assert idx == [0, 1, 64, 65, 128, 129, 192, 193]
    assert {i // 64 for i in idx} == {0, 1, 2, 3}


def test_run_concurrent_order_and_errors():
    out = batch.run_concurrent(lambda item, lane: {"x": item * item, "lane": lane}, list(range(10)), 3)
    assert [o["x"] for o in out] == [i * i for i in range(10)]
    assert {o["lane"] for o in out} <= {0, 1, 2}

    def bad(item, lane):
        if item == 4:
            raise RuntimeError("boom")
        return {}
    with pytest.raises(RuntimeError):
        batch.run_concurrent(bad, list(range(8)), 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        items = batch.shard(9, rank, world)                    # uneven: 5 + 4
        local = [{"index": i, "steps": 3 + i % 2, "res": 1e-15 * (i + 1)} for i in items]
        allres = batch.gather_results(local, ["index", "steps", "res"])
        tmax = batch.max_over_ranks(float(rank + 1))
        q.put((rank, [r["index"] for r in allres], [r["steps"] for r in allres], tmax))
    finally:
        dist.destroy_process_group()


def test_gather_and_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, idx, steps, tmax in got:
        assert idx == list(range(9))                           # every rank sees all results in order
        assert steps == [3 + i % 2 for i in range(9)]
        assert tmax == 2.0                                     # the slowest rank's time

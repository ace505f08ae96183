"""World-size-2 gloo tests of the multi-GPU host logic (CPU only): IPC handle
exchange ordering and the virtual-rank -> GPU partition the device kernels
assume (rank r on GPU r // (G/P), topology.py:99-100 style contiguity)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import moe as OM


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_09591_b200.layer import exchange_handles, rank_placement
    mine = bytes([rank * 16 + i for i in range(64)])
    allh = exchange_handles(mine, rank, world)
    ok = all(allh[q_ * 64:(q_ + 1) * 64] == bytes([q_ * 16 + i for i in range(64)])
             for q_ in range(world))
    # per-GPU count rows assembled over gloo == the global dedup histogram
    G, E, K, T_r = 8, 64, 6, 40
    rng = np.random.default_rng(5)
    logits = rng.standard_normal((G * T_r, E)).astype(np.float32)
    ids, _, _ = OM.route_topk(logits, K)
    plan = OM.DispatchPlan(ids, G, E)
    mine_ranks = rank_placement(G, world, rank)
    import torch
    rows = torch.tensor(plan.h[list(mine_ranks)], dtype=torch.int64)
    parts = [torch.empty_like(rows) for _ in range(world)]
    dist.all_gather(parts, rows)
    full = torch.cat(parts).numpy()
    q.put((rank, ok, np.array_equal(full, plan.h), list(mine_ranks)))
    dist.destroy_process_group()


def test_gloo_world2_handle_exchange_and_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [True, True]
    assert res[0][3] == [0, 1, 2, 3] and res[1][3] == [4, 5, 6, 7]


def test_rank_placement_rejects_uneven():
    from paper_2508_09591_b200.layer import rank_placement
    with pytest.raises(ValueError):
        rank_placement(8, 3, 0)

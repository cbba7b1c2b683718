"""CPU, world size 2 over gloo: the host-side logic of the one-rank-per-GPU
deployment, through the product's own host functions (the C ABI) — partition
ownership and tiling per rank, the replicated control plane staying identical
on every rank, the NCCL-id rendezvous, and bench.py's max-over-ranks timing."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import numpy as np
    import torch.distributed as dist

    import bench
    from paper_2402_13781_b200 import sparsim as S
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n_g, n_b, min_blk = 1_000_003, 16 * world, 2
        cfg = S.validate(S.SparsifierConfig(n=world, n_g=n_g, n_b=n_b, d=0.01, min_blk=min_blk))
        topo = S.build_topology(n_g, n_b, world, min_blk)
        k_t = [cfg.k // world] * world  # engine.cpp:75
        rng = np.random.default_rng(1000 + rank)
        for t in range(24):
            # this rank's plan (engine.cpp:125-131) through the C ABI
            part = S.rotate_to_partition_order(k_t, t, world)
            S.adjust_topology(topo, part, cfg.alpha, cfg.blk_move, cfg.min_blk, n_g)
            a = S.allocate_partition(topo, t, rank, n_g)
            # every rank must hold the same replicated control state
            states = [None] * world
            dist.all_gather_object(states, (topo.blk_part, topo.blk_pos, a.partition,
                                            a.range.st, a.range.end))
            parts = [s_[:2] for s_ in states]
            assert all(p == parts[0] for p in parts), (t, parts)
            owned = sorted((s_[3], s_[4], r) for r, s_ in enumerate(states))
            cursor = 0
            for st, end, _ in owned:  # ranges tile [0, n_g) disjointly
                assert st == cursor and end > st
                cursor = end
            assert cursor == n_g
            for r, s_ in enumerate(states):  # cyclic ownership (t % n + r) % n
                assert s_[2] == (t % world + r) % world
            # skewed per-rank counts, gathered in rank order (the count all-gather)
            mine = int(rng.integers(0, 3 * cfg.k // world))
            got = [None] * world
            dist.all_gather_object(got, mine)
            k_t = got
            g = S.gather_stats(k_t)
            assert g.k_prime == sum(k_t) and g.m_t == max(k_t)
        # NCCL-id rendezvous used by bench.py / tools/dist_check.py
        try:
            ids = [S.nccl_unique_id() if rank == 0 else None]
        except S.DeviceError:
            ids = [b"x" * 128 if rank == 0 else None]  # no NCCL transport on this host
        dist.broadcast_object_list(ids, src=0)
        assert len(ids[0]) == 128
        # bench.py's whole-job timing is the max over ranks
        out = bench.max_over_ranks([1.0 + rank, 5.0 - rank], dist)
        assert out == [float(world), 5.0]
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
        raise


@pytest.mark.parametrize("world", [2])
def test_two_rank_host_logic_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert results == {r: "ok" for r in range(world)}, results
    assert all(p.exitcode == 0 for p in procs)

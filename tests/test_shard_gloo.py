"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the N > 1 host path:
the subband partition, the W broadcast and the max-over-ranks timing
reduction.  The data path has no collective; the oracle is
used here only to show that sharded results equal the unsharded ones."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bf_synth as syn
        import oracle
        from paper_1810_11451_b200 import shard
        wl = syn.workload("c4")
        tags_all = syn.subband_tags(wl.seed, np.arange(n), wl.n_groups)
        ids = shard.subband_shard(tags_all, rank, world)
        # W broadcast: only rank 0 draws it
        W = torch.zeros((wl.n_groups, 64, 36), dtype=torch.complex64)
        if rank == 0:
            W.copy_(torch.from_numpy(syn.precoders(wl.seed, 0, wl.n_groups, 64, 36, wl.w_norm)))
        shard.broadcast_precoders(W)
        # this rank's share of the work (oracle stands in for the GPU on CPU)
        S = syn.qam_symbols(wl.seed, 0, ids, 36, 60, 64)
        R, _, _ = oracle.beamform(W.numpy(), S, tags_all[ids])
        mx = shard.max_over_ranks(float(rank + 1))
        tot = shard.sum_over_ranks(float(len(ids)))
        q.put((rank, ids, R, W.numpy(), mx, tot))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


@pytest.mark.parametrize("world", [2, 3])
def test_subband_sharding_gloo(world):
    import bf_synth as syn
    import oracle
    n = 1200
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_ids = np.concatenate([o[1] for o in out])
    assert np.array_equal(np.sort(all_ids), np.arange(n))          # disjoint cover
    sizes = [len(o[1]) for o in out]
    assert max(sizes) - min(sizes) <= 1                            # balanced to one block
    wl = syn.workload("c4")
    tags = syn.subband_tags(wl.seed, np.arange(n), wl.n_groups)
    for o in out:                                                  # few subbands per rank
        assert len(np.unique(tags[o[1]])) <= -(-55 // world) + 1
        assert np.array_equal(o[3], out[0][3])                     # W replicated bitwise
        assert o[4] == float(world) and o[5] == float(n)
    W = syn.precoders(wl.seed, 0, wl.n_groups, 64, 36, wl.w_norm)
    S = syn.qam_symbols(wl.seed, 0, np.arange(n), 36, 60, 64)
    R_all, _, _ = oracle.beamform(W, S, tags, n_threads=4)
    for o in out:                                                  # sharding never changes results
        assert np.array_equal(o[2].view(np.uint32), R_all[o[1]].view(np.uint32))


def test_even_range_and_chunk_shard():
    from paper_1810_11451_b200 import shard
    for n, w in [(770, 8), (100_000, 3), (5, 8)]:
        parts = [shard.even_range(n, r, w) for r in range(w)]
        assert sum(c for _, c in parts) == n
        assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(w - 1))
        assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    first, cnt = shard.chunk_shard(7, 4096, 1, 4)
    assert (first, cnt) == (7 * 4096 + 1024, 1024)
    with pytest.raises(ValueError):
        shard.even_range(10, 3, 3)


def _window_worker(rank, world, port, n_chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bf_synth as syn
        from paper_1810_11451_b200 import shard
        wins = shard.window_shard(n_chunks, 8, rank, world)
        mine = [c for w in wins for c in w]
        fc = syn.cell_flows(syn.workload("c5").seed, 8)
        work = float(sum(int(fc[c % 8]) + 64 for c in mine))      # bytes per block ~ f + 64
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        q.put((rank, wins, allv, shard.max_over_ranks(work), shard.sum_over_ranks(work)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_c5_window_dealing_gloo(world):
    """c5: whole 8-chunk windows dealt round-robin (window w -> rank w mod world): every chunk
    exactly once, each window one chunk of every cell, every rank the same per-cell mix, so
    the per-rank work (sum of f + 64 over its chunks) is equal."""
    n_chunks = 2048
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_window_worker, args=(r, world, port, n_chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered = out[0][2]
    assert all(o[2] == gathered for o in out)                      # every rank agrees
    allc = np.concatenate([np.asarray(g) for g in gathered])
    assert np.array_equal(np.sort(allc), np.arange(n_chunks))      # disjoint cover
    for rank, wins, _, mx, tot in out:
        for w in wins:
            assert len(w) == 8 and sorted(c % 8 for c in w) == list(range(8))   # one per cell
            assert w[0] // 8 % world == rank
        cells = np.bincount(np.asarray([c for w in wins for c in w]) % 8, minlength=8)
        assert (cells == n_chunks // 8 // world).all()              # same per-cell mix
        assert mx * world == tot                                    # perfectly balanced


def test_window_shard_ragged():
    from paper_1810_11451_b200 import shard
    for n_chunks, world in [(2048, 8), (100, 3), (5, 4), (1, 2)]:
        got = [c for r in range(world) for w in shard.window_shard(n_chunks, 8, r, world) for c in w]
        assert sorted(got) == list(range(n_chunks))
    assert shard.window_shard(5, 8, 1, 4) == []
    with pytest.raises(ValueError):
        shard.window_shard(10, 0, 0, 1)

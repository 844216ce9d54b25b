"""World-size-2 gloo tests of the multi-rank host logic used by bench.py --gpus N (CPU only)."""
import importlib.util
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load_dist():
    # import the module by path: the package __init__ loads the CUDA library, which is not needed here
    spec = importlib.util.spec_from_file_location("pscwin_dist", os.path.join(ROOT, "paper_2407_02109_b200", "dist.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    d = _load_dist()
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = d.env_rank_world()
    lo, hi = d.shard_range(8, w, r)
    # per-rank "step times": the job time is the max over ranks; images are counted once each
    t = d.max_over_ranks(1.5 + rank)
    n = d.sum_over_ranks(hi - lo)
    out[rank] = (r, w, lr, lo, hi, t, n)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_reduce():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][:3] == (0, 2, 0) and out[1][:3] == (1, 2, 1)
    assert (out[0][3], out[0][4]) == (0, 4) and (out[1][3], out[1][4]) == (4, 8)
    assert out[0][5] == out[1][5] == 2.5          # max over ranks
    assert out[0][6] == out[1][6] == 8            # every image processed exactly once


@pytest.mark.parametrize("n,world", [(8, 1), (8, 3), (1, 2), (13, 4)])
def test_shard_range_partition(n, world):
    d = _load_dist()
    seen = []
    for r in range(world):
        lo, hi = d.shard_range(n, world, r)
        assert 0 <= lo <= hi <= n
        seen.extend(range(lo, hi))
    assert seen == list(range(n))
    with pytest.raises(ValueError):
        d.shard_range(n, world, world)


def test_single_process_reduce_is_identity():
    d = _load_dist()
    assert d.max_over_ranks(3.25) == 3.25


# ------------------------------------------------------------------ window-row bands (host logic of §8(e))
def _band_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    d = _load_dist()
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = d.TorchDistExchange()
    # ring: rank g receives rank g-1's bytes (rank 0 the last rank's)
    send = torch.full((6,), 10 + rank, dtype=torch.uint8)
    recv = torch.zeros(6, dtype=torch.uint8)
    ex.ring(send, recv)
    # all-gather in rank order
    rec = torch.arange(4, dtype=torch.uint8) + 100 * rank
    recs = torch.zeros(4 * world, dtype=torch.uint8)
    ex.allgather(rec, recs)
    # halo: rank 0 has no previous neighbour, the last rank no next one; sizes agree pairwise (3 down, 5 up)
    sp = torch.full((3 if rank > 0 else 0,), 30 + rank, dtype=torch.uint8)
    sn = torch.full((5 if rank < world - 1 else 0,), 50 + rank, dtype=torch.uint8)
    rp = torch.zeros(5 if rank > 0 else 0, dtype=torch.uint8)
    rn = torch.zeros(3 if rank < world - 1 else 0, dtype=torch.uint8)
    ex.halo(sp, sn, rp, rn)
    out[rank] = (recv.tolist(), recs.tolist(), rp.tolist(), rn.tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_exchange_gloo(world):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_band_worker, args=(world, port, out), nprocs=world, join=True)
    for g in range(world):
        recv, recs, rp, rn = out[g]
        assert recv == [10 + (g - 1) % world] * 6
        assert recs == [v + 100 * r for r in range(world) for v in range(4)]
        assert rp == ([50 + g - 1] * 5 if g > 0 else [])
        assert rn == ([30 + g + 1] * 3 if g < world - 1 else [])


@pytest.mark.parametrize("H,w,world", [(256, 16, 8), (64, 16, 4), (28, 8, 3), (34, 8, 3), (32, 8, 1), (36, 8, 4)])
def test_band_rows_cover_whole_window_rows(H, w, world):
    d = _load_dist()
    rows = d.band_rows(H, w, world)
    assert rows[0][0] == 0 and rows[-1][1] == H and len(rows) == world
    for (a, b), (c, _) in zip(rows, rows[1:]):
        assert b == c and a % w == 0 and b % w == 0 and b > a
    assert all(r1 - r0 >= w for r0, r1 in rows)      # every band can serve a halo of up to w - 1 rows
    with pytest.raises(ValueError):
        d.band_rows(H, w, H // w + 1)


def test_band_rows_ragged_tail_joins_last_band():
    # a ragged last band shorter than the halo it must send (H = 34, w = 8, 3 ranks) is never produced
    d = _load_dist()
    assert d.band_rows(34, 8, 3) == [(0, 16), (16, 24), (24, 34)]
    with pytest.raises(ValueError):
        d.band_rows(20, 8, 3)                          # 2 whole window rows (+ 4 ragged) cannot feed 3 ranks

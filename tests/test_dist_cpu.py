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

"""Host-side multi-GPU logic (row a-7) on the CPU: shard arithmetic and a
world_size-2 gloo all-gather that must reassemble the full NCHW Out from the
per-rank slabs.  The slabs are computed by the oracle here (test
infrastructure); on the GPU box they come from libconv.so (tests/test_parity.py
checks that n-shards are bit-identical to slices of the 1-GPU result)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2101_09808_b200.inputs import Shape, make_inputs
from paper_2101_09808_b200.shard import gather, local_inputs, shard


def test_shard_ranges_cover_and_partition():
    sh = Shape(N=256, K=256, C=256, H=14, W=14, R=3, S=3)
    for world in (1, 2, 4, 8):
        specs = [shard(sh, world, r) for r in range(world)]
        assert specs[0].start == 0 and specs[-1].stop == sh.N
        for a, b in zip(specs, specs[1:]):
            assert a.stop == b.start
        assert all(s.local.N == sh.N // world for s in specs)


def test_shard_auto_picks_k_for_small_batch():
    sh = Shape(N=1, K=64, C=32, H=8, W=8, R=3, S=3)
    s = shard(sh, 4, 1)
    assert s.dim == "k" and (s.start, s.stop) == (16, 32) and s.local.K == 16


def test_shard_keeps_stride_and_input_extents():
    sh = Shape.strided(8, 64, 32, 29, 29, 3, 3, 2)
    for dim, world in (("n", 4), ("k", 2)):
        loc = shard(sh if dim == "n" else Shape.strided(1, 64, 32, 29, 29, 3, 3, 2), world, 1, dim=dim).local
        assert (loc.U, loc.Hin, loc.Win, loc.H, loc.W) == (2, 29, 29, 14, 14)


def test_shard_errors():
    with pytest.raises(ValueError):
        shard(Shape(N=3, K=4, C=1, H=1, W=1, R=1, S=1), 2, 0, dim="n")
    with pytest.raises(ValueError):
        shard(Shape(N=2, K=4, C=1, H=1, W=1, R=1, S=1), 2, 0, dim="k")
    with pytest.raises(ValueError):
        shard(Shape(N=2, K=4, C=1, H=1, W=1, R=1, S=1), 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape_t, dim, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = Shape(*shape_t)
        inp, ker = make_inputs(sh, seed=3)
        spec = shard(sh, world, rank, dim=dim)
        li, lk = local_inputs(spec, inp, ker)
        slab = torch.from_numpy(oracle.conv_eq1(li.numpy(), lk.numpy()).astype(np.float32))
        full = gather(slab, spec)
        if rank == 0:
            result_q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape_t,dim", [((4, 6, 3, 5, 7, 3, 3), "n"), ((1, 8, 3, 5, 6, 3, 2), "k")])
def test_gloo_world2_gather_reassembles_out(shape_t, dim):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape_t, dim, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sh = Shape(*shape_t)
    inp, ker = make_inputs(sh, seed=3)
    ref = oracle.conv_eq1(inp.numpy(), ker.numpy()).astype(np.float32)
    assert full.shape == ref.shape
    assert np.array_equal(full, ref)

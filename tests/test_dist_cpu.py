"""Multi-GPU host logic on CPU: bin ownership, tile pack/unpack and the
rank-0 gather (torch.distributed, gloo, world_size 2 and 4), checked against
a single-process frame from the C restatement."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import bindings
import shard_host as vdist
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import default_params


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_ownership_partitions_bins(world):
    bx, by = 60, 34
    seen = np.zeros((by, bx), dtype=int)
    for r in range(world):
        for x, y in vdist.owned_bins(bx, by, r, world):
            seen[y, x] += 1
        # libveil's host-side count agrees with the Python rule
        assert veil.shard_tile_count(bx, by, r, world) == len(vdist.owned_bins(bx, by, r, world))
    assert (seen == 1).all()
    counts = [len(vdist.owned_bins(bx, by, r, world)) for r in range(world)]
    assert max(counts) - min(counts) <= 1 + bx // world  # interleave is balanced


def test_pack_unpack_roundtrip_ragged():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 255, (75, 101, 4), dtype=np.uint8)
    mask = rng.integers(0, 2, (75, 101), dtype=np.uint8)
    out_i = np.zeros_like(img)
    out_m = np.zeros_like(mask)
    for r in range(3):
        vdist.unpack_tiles(vdist.pack_tiles(img, mask, r, 3), out_i, out_m, r, 3)
    assert np.array_equal(out_i, img) and np.array_equal(out_m, mask)


def _worker(rank, world, port, ret):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    arr = veil.Scene.synthetic("random_soup", 9, 160, 96).arrays()
    # each rank "renders" the frame with the restatement and keeps its bins
    o = bindings.oracle_render(arr, default_params(), names={"image", "mask"})
    img = o["image"].reshape(96, 160, 4)
    mask = o["mask"].reshape(96, 160)
    bx, by = 5, 3
    cap = vdist.max_tiles(bx, by, world)
    tiles = torch.from_numpy(vdist.pack_tiles(img, mask, rank, world, cap))
    bufs = vdist.gather_frame(tiles, rank, world)
    if rank == 0:
        out_i = np.zeros_like(img)
        out_m = np.zeros_like(mask)
        for r in range(world):
            vdist.unpack_tiles(bufs[r].numpy(), out_i, out_m, r, world)
        ret[0] = int(np.array_equal(out_i, img) and np.array_equal(out_m, mask))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_gather_reassembles_frame(world):
    ctx = mp.get_context("spawn")
    ret = ctx.Array("i", [0])
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert ret[0] == 1

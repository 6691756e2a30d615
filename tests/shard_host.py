"""Host twins of the screen-space sharding layout. TEST HELPER.

tests/test_dist_cpu.py uses these to check, with gloo processes on CPU, the
tile layout and the gather that bench.py's NCCL path performs on the GPU.

Bins are interleaved over ranks with owner(bx, by) = (bx + 3*by) mod world
(the same rule libveil's kernels apply, include/veil_cuda.h). Every rank
replicates setup and binning (so visible indices stay global and bin lists
are bit-exact), rasterizes only its bins, packs its finished 32x32 tiles
(4096 B RGBA8 + 1024 B invalid mask each) and rank 0 gathers them over NCCL
(NVLink) and unpacks them into the full frame.

The packing/unpacking used on the GPU is libveil's k_tile_copy
(veil_shard_pack_tiles_device / veil_shard_unpack_tiles_device); the numpy
versions below define the same layout for host buffers and tests.
"""
import numpy as np

TILE = 32
TILE_BYTES = TILE * TILE * 4 + TILE * TILE


def owner(bx, by, world):
    return (bx + 3 * by) % world


def owned_bins(bins_x, bins_y, rank, world):
    """Row-major list of (bx, by) owned by rank."""
    return [(x, y) for y in range(bins_y) for x in range(bins_x) if owner(x, y, world) == rank]


def max_tiles(bins_x, bins_y, world):
    return max(len(owned_bins(bins_x, bins_y, r, world)) for r in range(world))


def pack_tiles(rgba, mask, rank, world, capacity_tiles=None):
    """Host twin of k_tile_copy(pack): rgba (H, W, 4) u8, mask (H, W) u8."""
    h, w = mask.shape
    bx, by = (w + TILE - 1) // TILE, (h + TILE - 1) // TILE
    bins = owned_bins(bx, by, rank, world)
    n = capacity_tiles if capacity_tiles is not None else len(bins)
    out = np.zeros((n, TILE_BYTES), dtype=np.uint8)
    for i, (x, y) in enumerate(bins):
        px, py = x * TILE, y * TILE
        tw, th = min(TILE, w - px), min(TILE, h - py)
        t = np.zeros((TILE, TILE, 4), dtype=np.uint8)
        m = np.zeros((TILE, TILE), dtype=np.uint8)
        t[:th, :tw] = rgba[py:py + th, px:px + tw]
        m[:th, :tw] = mask[py:py + th, px:px + tw]
        out[i, :4096] = t.reshape(-1)
        out[i, 4096:] = m.reshape(-1)
    return out.reshape(-1)


def unpack_tiles(tiles, rgba, mask, rank, world):
    """Host twin of k_tile_copy(unpack): writes rank's tiles into the frame."""
    h, w = mask.shape
    bx, by = (w + TILE - 1) // TILE, (h + TILE - 1) // TILE
    tiles = np.asarray(tiles, dtype=np.uint8).reshape(-1, TILE_BYTES)
    for i, (x, y) in enumerate(owned_bins(bx, by, rank, world)):
        px, py = x * TILE, y * TILE
        tw, th = min(TILE, w - px), min(TILE, h - py)
        rgba[py:py + th, px:px + tw] = tiles[i, :4096].reshape(TILE, TILE, 4)[:th, :tw]
        mask[py:py + th, px:px + tw] = tiles[i, 4096:].reshape(TILE, TILE)[:th, :tw]


def gather_frame(tiles_tensor, rank, world, dst=0):
    """torch.distributed gather of equally sized tile buffers to dst.

    tiles_tensor: uint8 tensor of max_tiles * TILE_BYTES (padded). Returns the
    list of per-rank buffers on dst, None elsewhere. NCCL (GPU tensors) or
    gloo (CPU tensors), whichever backend the process group uses.
    """
    import torch
    import torch.distributed as dist

    if rank == dst:
        bufs = [torch.empty_like(tiles_tensor) for _ in range(world)]
        dist.gather(tiles_tensor, bufs, dst=dst)
        return bufs
    dist.gather(tiles_tensor, None, dst=dst)
    return None

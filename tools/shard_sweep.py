"""Per-rank frame time of a bin-interleaved shard, measured on one GPU.

    python tools/shard_sweep.py [workload ...]

For G = 1, 2, 4, 8 it renders shard (0, G) -- rank 0's bins of a G-way split,
including the replicated cull/compaction -- and prints the median device ms
per frame (CUDA events). On a G-GPU node every rank does this work at the
same time (the bins are interleaved, so their loads are close), so
ms(1) / ms(G) bounds the device-side speed-up before the framebuffer gather.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_13364_b200 import veil  # noqa: E402

SEEDS = {"stack64k": 2, "tiny4m": 4, "mixed16m": 5}
for name in sys.argv[1:] or ["stack64k", "tiny4m", "mixed16m"]:
    sc = veil.Scene.workload(name, SEEDS[name])
    base = None
    for g in (1, 2, 4, 8):
        ms = []
        for r in range(g):  # every rank's share, so the slowest rank is visible
            for _ in range(3):
                veil.render_device(sc, None, (r, g))
            sts = [veil.render_device(sc, None, (r, g)) for _ in range(10)]
            ms.append((statistics.median(s.total_ms for s in sts),
                       {k: statistics.median(getattr(s, k) for s in sts)
                        for k in ("setup_ms", "binning_ms", "low_raster_ms", "hi_raster_ms", "shade_ms")}))
        worst, stages = max(ms, key=lambda x: x[0])
        base = base or worst
        print(f"{name:9s} G={g}: slowest rank {worst:.3f} ms/frame (ranks {min(m[0] for m in ms):.3f}..{worst:.3f}), "
              f"speed-up bound {base / worst:.2f}x  stages " +
              " ".join(f"{k[:-3]} {v:.3f}" for k, v in stages.items()), flush=True)

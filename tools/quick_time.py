import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import default_params
for name, seed in [("stack64k", 2), ("tiny4m", 4)]:
    t = time.time(); sc = veil.Scene.workload(name, seed); print(name, "gen", time.time() - t, flush=True)
    for i in range(5):
        st = veil.render_device(sc)
    t = time.perf_counter()
    for i in range(20):
        veil.render_device(sc)
    print(name, "wall_ms_per_frame", (time.perf_counter() - t) / 20 * 1e3, flush=True)
    print(name, "ms", st.total_ms, "shade", st.shade_ms, "setup", st.setup_ms, "bin", st.binning_ms, "low", st.low_raster_ms, "high", st.hi_raster_ms,
          "frags", st.fragments, "samples", st.samples, "thb", st.tri_half_blocks, "pairs", st.bin_pairs,
          "vis", st.visible_quads, "bins", st.bins_empty, st.bins_low, st.bins_high, st.bins_propagated, flush=True)

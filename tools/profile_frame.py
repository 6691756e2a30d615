"""Warm frames of a workload for ncu: python tools/profile_frame.py stack64k [frames] [rank world]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_13364_b200 import veil
name = sys.argv[1] if len(sys.argv) > 1 else "stack64k"
seed = {"stack64k": 2, "tiny4m": 4, "mixed16m": 5}[name]
sc = veil.Scene.workload(name, seed)
shard = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else None
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    st = veil.render_device(sc, None, shard)
print(name, st.total_ms, st.low_raster_ms, st.hi_raster_ms)

"""A/B timing of libveil builds: python tools/ab_time.py lib1.so lib2.so ...
Each build renders stack64k and tiny4m in a fresh process; prints medians of
20 frames per stage (CUDA events), interleaving builds over 2 rounds."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, statistics, json
sys.path.insert(0, os.environ["ROOT"])
from paper_2405_13364_b200 import veil
out = {}
for name in os.environ.get("AB_WORKLOADS", "stack64k,tiny4m").split(","):
    if name == "boxes1080":  # C3's scene (one orbit camera: the arrays' own)
        sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
        from common import boxes_arrays
        sc = veil.Scene.from_arrays(boxes_arrays(1920, 1080))
    else:
        sc = veil.Scene.workload(name, {"stack64k": 2, "tiny4m": 4, "mixed16m": 5}[name])
    for i in range(5): veil.render_device(sc)
    st = [veil.render_device(sc) for i in range(20)]
    med = lambda f: statistics.median(f(s) for s in st)
    out[name] = {"total": med(lambda s: s.total_ms), "shade": med(lambda s: s.shade_ms),
                 "setup": med(lambda s: s.setup_ms), "bin": med(lambda s: s.binning_ms),
                 "low": med(lambda s: s.low_raster_ms), "high": med(lambda s: s.hi_raster_ms)}
print(json.dumps(out))
'''
libs = sys.argv[1:]
res = {l: [] for l in libs}
for rnd in range(2):
    for l in libs:
        env = dict(os.environ, VEIL_LIB=os.path.abspath(l), ROOT=ROOT)
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        if p.returncode:
            print(l, "FAILED", p.stderr[-500:]); continue
        res[l].append(json.loads(p.stdout.strip().splitlines()[-1]))
for l in libs:
    for w in os.environ.get("AB_WORKLOADS", "stack64k,tiny4m").split(","):
        rows = [r[w] for r in res[l]]
        if not rows: continue
        keys = rows[0].keys()
        print(f"{os.path.basename(l):28s} {w:9s} " + " ".join(f"{k} {min(r[k] for r in rows):.4f}" for k in keys))

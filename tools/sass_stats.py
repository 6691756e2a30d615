"""Per-kernel SASS statistics of libveil.so: instruction count, local-memory
ops (LDL/STL), FP64 ops, shared/global loads. usage: tools/sass_stats.py [filter]"""
import re, subprocess, sys, collections
so = "paper_2405_13364_b200/libveil.so"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None; stats = collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); stats[cur] = collections.Counter(); continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        op = m.group(2).split(".")[0]
        stats[cur]["inst"] += 1
        if op in ("LDL", "STL"): stats[cur]["local"] += 1
        if op.startswith("D") and op in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"): stats[cur]["fp64"] += 1
        if op in ("LDS", "STS"): stats[cur]["smem"] += 1
        if op in ("LDG", "STG"): stats[cur]["gmem"] += 1
        if op in ("UBLKCP", "UTMALDG", "SYNCS"): stats[cur]["bulk"] += 1
for k, v in stats.items():
    if flt in k:
        print(f"{v['inst']:6d} inst {v['local']:4d} local {v['fp64']:5d} fp64 {v['smem']:4d} smem {v['gmem']:4d} gmem "
              f"{v['bulk']:3d} bulk/mbar  {k[:90]}")

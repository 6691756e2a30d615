"""Aggregate an ncu source page (cuda,sass) per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilt = sys.argv[3:]  # extra ncu filter args, e.g. --launch-skip 4 --launch-count 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"] + kfilt,
                     capture_output=True, text=True).stdout
cur_file = None; agg = collections.defaultdict(lambda: [0, 0, 0, "", 0]); hdr = None; cur_line = None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": cur_file = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None: continue
    # rows: line-level rows have Line No + source; sass rows have empty line no
    if row[0] and row[0].isdigit():
        cur_line = (cur_file, int(row[0])); agg[cur_line][3] = row[1].strip()[:70]
        try:
            i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_e = hdr.index("Instructions Executed")
            agg[cur_line][0] += int(row[i_s] or 0); agg[cur_line][1] += int(row[i_e] or 0)
            i_t = hdr.index("Thread Instructions Executed"); agg[cur_line][4] += int(row[i_t] or 0)
        except (ValueError, IndexError): pass
tot_s = sum(v[0] for v in agg.values()) or 1; tot_e = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:5d} stall {100*v[0]/tot_s:5.1f}%  inst {100*v[1]/tot_e:5.1f}%  thr {v[4]/max(v[1],1):4.1f}  {v[3]}")

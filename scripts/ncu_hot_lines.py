#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples for one kernel of an .ncu-rep (needs
-lineinfo and --import-source on).   python scripts/ncu_hot_lines.py rep.ncu-rep k_solve [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, recs, seen_fn = None, None, [], set()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file, hdr = r[1].split("/")[-1], None
        continue
    if r[0] == "Function Name":
        fn = r[1][:60]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        i_s, i_i, i_t = hdr.index("# Samples"), hdr.index("Instructions Executed"), hdr.index("Avg. Threads Executed")
        try:
            samples, inst = int(r[i_s] or 0), int(r[i_i] or 0)
        except ValueError:
            continue
        if samples or inst:
            recs.append((samples, inst, cur_file, r[0], r[1].strip()[:100], r[i_t]))
tot = sum(r[0] for r in recs) or 1
toti = sum(r[1] for r in recs) or 1
print(f"kernel {kern}: total samples {tot}, total warp instructions {toti}")
for s, i, f, ln, src, thr in sorted(recs, reverse=True)[:top]:
    print(f"{s / tot:6.1%} samp {i / toti:6.1%} inst thr {thr:>3}  {f}:{ln:>4}  {src}")

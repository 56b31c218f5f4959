"""Per-CUDA-source-line digest of an ncu report (stall samples, instructions,
shared wavefronts) from `ncu -i rep --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
fname, hdr = None, None
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    try:
        s = int(r[4] or 0)
        ie = int(r[7] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg[key]
    a[0] += s
    a[1] += ie
    if "L1 Wavefronts Shared" in hdr:
        try:
            a[2] += int(r[hdr.index("L1 Wavefronts Shared")] or 0)
        except ValueError:
            pass
    a[3] = r[1].strip()[:80]
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% stall {100 * v[1] / toti:5.1f}% inst sh={v[2]:>9} {f}:{ln} | {v[3]}")

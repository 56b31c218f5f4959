"""SASS evidence for the hot kernels of libshearlet_b200.so: per kernel the
static instruction mix (FP64 math, shared / global memory, warp shuffles,
barriers, TMA) from `cuobjdump -sass`, written as a markdown table.
    python tools/sass_summary.py [lib] [out.md]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1402_5670_b200", "libshearlet_b200.so")
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r2_sass_summary.md")
HOT = [r"k2_rows_fusedILi512ELb1E7double2", r"k2_cols_decILi512E7double2", r"k2_cols_recILi512E7double2",
       r"k3s_decILi192E", r"k3s_midILi192ELi0ELb1E", r"k3s_recILi192E", r"k2_rows_fusedILi512ELb1E6float2",
       r"k3s_midILi128ELi0ELb1E"]
OPS = ["DFMA", "DADD", "DMUL", "FFMA", "LDS", "STS", "LDGSTS", "LDG", "STG", "SHFL", "BAR", "UTMALDG", "UTMASTG",
       "LDL", "STL"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
rows = []
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not any(re.search(h, name) for h in HOT):
        continue
    cnt = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9]+)", line)
        if m:
            cnt[m.group(2)] += 1
    rows.append((name, cnt))
with open(out, "w") as fh:
    fh.write("# SASS instruction mix of the hot kernels (static counts, `cuobjdump -sass`)\n\n")
    fh.write(f"library: `{os.path.relpath(lib, ROOT)}` (sm_100a). LDL/STL = spills; SHFL = the warp-shuffle mirror\n"
             "pairs of the r2c split (`mirror_pairs_shfl`); LDGSTS = cp.async tile staging.\n\n")
    fh.write("| kernel | " + " | ".join(OPS) + " | total |\n|---|" + "---|" * (len(OPS) + 1) + "\n")
    for name, cnt in rows:
        fh.write(f"| `{name[:60]}` | " + " | ".join(str(cnt.get(o, 0)) for o in OPS) + f" | {sum(cnt.values())} |\n")
print(open(out).read())

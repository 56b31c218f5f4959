"""Summarise ncu output into the tracked profiles/ files.

    python tools/ncu_summary.py full   <report.ncu-rep> <out.csv>
        one row per captured kernel: duration, grid/block/regs, occupancy,
        FP64/L1/L2/DRAM utilisation, DRAM bytes, top-4 stall reasons.
    python tools/ncu_summary.py launches <launches.csv> <out.md>
        per-kernel launch count, mean duration and share of the captured
        launches (the `--metrics gpu__time_duration.sum` launch list).
"""
import collections
import csv
import io
import subprocess
import sys

COLS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]
STALL = "smsp__average_warps_issue_stalled_"


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    stall_cols = [i for i, n in enumerate(h) if n.startswith(STALL) and n.endswith("_per_issue_active.ratio")]
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel"] + [c for c in COLS if c in h] + ["top_stalls"])
        for r in rows[2:]:
            vals = [f"{r[h.index(c)]} {units[h.index(c)]}".strip() for c in COLS if c in h]
            st = sorted(((float(r[i] or 0), h[i][len(STALL):].replace("_per_issue_active.ratio", "")) for i in stall_cols),
                        reverse=True)[:4]
            w.writerow([r[h.index("Kernel Name")][:40]] + vals + [str([(round(v, 3), n) for v, n in st])])
    print(f"wrote {out}")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    t, n = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
        k = r[ki].split(">(")[0].replace("void ", "").replace("(int)", "") + ">"
        t[k] += float(r[vi].replace(",", "")) * scale
        n[k] += 1
    tot = sum(t.values())
    with open(out, "w") as fh:
        fh.write(f"# launch list summary: {path.split('/')[-1]}\n\n")
        fh.write("cold-cache, serialised ncu launches (`--metrics gpu__time_duration.sum --clock-control none`);\n")
        fh.write("compare SHARES with bench.py's live per-pass timing, not absolute times.\n\n")
        fh.write("| kernel | launches | mean us | share |\n|---|---|---|---|\n")
        for k in sorted(t, key=lambda k: -t[k]):
            fh.write(f"| `{k}` | {n[k]} | {t[k] / n[k]:.1f} | {100 * t[k] / tot:.1f} % |\n")
        fh.write(f"\ntotal captured: {tot:.0f} us over {sum(n.values())} launches\n")
    print(f"wrote {out}")


# pass names bench.py reports -> kernel whose grid y counts the bands of a launch
PASS_KERNEL = {"f2_rows_fused": "k2_rows_fused", "f3_rows_fused": "k2_rows_fused",
               "f2_cols_dec": "k2_cols_dec", "f2_cols_rec": "k2_cols_rec",
               "f2_rows_c2r_thr": "k2_rows_c2r", "f3_axis1": "k3_lines_contig",
               "f3s_dec": "k3s_dec", "f3s_mid": "k3s_mid", "f3s_rec": "k3s_rec",
               "f3g_dec": "k3g_dec", "f3g_rec": "k3g_rec"}
# kernels whose grid y is not the band count of the launch (band groups /
# in-kernel band loops): bands per launch of the capture drivers
# (tools/prof3d.py: a 12-band shard in one chunk; tools/prof2d.py: a lone
# 512^2 frame, all 49 bands in one chunk)
BANDS_OVERRIDE = {"k3s_dec": 12, "k3s_rec": 12, "k3g_dec": 12, "k3g_rec": 12, "k2_cols_dec": 49, "k2_cols_rec": 49}


def traffic(rep, out, config):
    """DRAM bytes per band of each pass's kernel from one `ncu --set full`
    capture (cold caches: ncu flushes between replays), merged into the
    JSON bench.py reads for roofline.traffic (profiles/traffic.json)."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    col = lambda r, name: float(r[h.index(name)].replace(",", "")) * scale.get(units[h.index(name)], 1)
    per_kernel = {}
    for r in rows[2:]:
        k = r[h.index("Kernel Name")].split("<")[0].replace("void ", "")
        gy = BANDS_OVERRIDE.get(k, int(r[h.index("launch__grid_dim_y")]))
        b = col(r, "dram__bytes_read.sum") + col(r, "dram__bytes_write.sum")
        per_kernel.setdefault(k, []).append(b / max(gy, 1))
    doc = json.load(open(out)) if os.path.exists(out) else {}
    entry = {}
    for pname, k in PASS_KERNEL.items():
        if k in per_kernel and pname.startswith("f3" if config.startswith("3d") else "f2"):
            v = per_kernel[k]
            entry[pname] = {"dram_bytes_per_band": sum(v) / len(v), "launches_captured": len(v)}
    entry["source"] = os.path.basename(rep)
    doc[config] = entry
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(f"wrote {out}: {config} {entry}")


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])

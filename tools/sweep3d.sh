#!/bin/bash
# 3D band-group sweep (SLB_G3) through bench.py; usage: tools/sweep3d.sh [config] ["G list"]
cfg=${1:-3d192}
for g in ${2:-1 2 4 8}; do
  out=$(SLB_G3=$g timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
  python - "$g" "$out" <<'PY'
import json, sys
g, line = sys.argv[1:3]
try:
    d = json.loads(line)
    k = {n: round(v["ms_total"] / max(1, v["launches"]), 4) for n, v in d["kernels"].items()}
    print(f"G3={g} value={d['value']:.2f} e2e={d['e2e']['value']:.2f} frac={d['path_roofline']['frac']:.3f} ms/launch={k}", flush=True)
except Exception:
    print(f"G3={g} failed: {line[:300]}")
PY
done

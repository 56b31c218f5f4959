#!/bin/bash
# Sweep the 2D launch knobs (band group G, chunk C, streams) through bench.py.
# usage: tools/sweep2d.sh [config] ["streams list"] ["G list"] ["C list"]
cfg=${1:-2d512}
for st in ${2:-4 8}; do for g in ${3:-2 4 7}; do for c in ${4:-14 28}; do
  out=$(SLB_STREAMS=$st SLB_GROUP=$g SLB_CHUNK=$c timeout 300 python bench.py --config $cfg --steps 30 --no-cpu-baseline 2>/dev/null | tail -1)
  python - "$st" "$g" "$c" "$out" <<'PY'
import json, sys
st, g, c, line = sys.argv[1:5]
try:
    d = json.loads(line)
    print(f"streams={st} G={g} C={c} value={d['value']:.1f} e2e={d['e2e']['value']:.1f} path_frac={d['path_roofline']['frac']:.3f}", flush=True)
except Exception as e:
    print(f"streams={st} G={g} C={c} failed: {line[:200]}")
PY
done; done; done

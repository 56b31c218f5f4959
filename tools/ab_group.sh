#!/bin/bash
# A/B of the concurrent band group default (r1o: G = 28 where it fits the chunk)
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for g in 14 ""; do for c in 2d512 2d256; do
  out=$(env ${g:+SLB_GROUP=$g} timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "G=${g:-default} $c $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")"
done; done; done
timeout 300 python bench.py --config 2d1024x64 --steps 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2d1024x64', round(d['value'],1), round(d['e2e']['value'],1))"

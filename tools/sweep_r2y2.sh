#!/bin/bash
cd "$(dirname "$0")/.."
run() { env "$@" python bench.py --no-3d --no-cpu-baseline --steps 60 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value']), round(d['e2e']['value']))"; }
for i in 1 2; do
run SLB_X=0
run SLB_LOCKSTEP_FRAMES=4
run SLB_GROUP=49 SLB_CHUNK=49
run SLB_LOCKSTEP_FRAMES=4 SLB_GROUP=49 SLB_CHUNK=49
done

#!/bin/bash
# 2D 512^2 x 8 device batch: lock-step frames per group x band group
cd "$(dirname "$0")/.."
run() { env "$@" python bench.py --no-3d --no-cpu-baseline --steps 40 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value']), round(d['e2e']['value']))"; }
run SLB_X=0
run SLB_LOCKSTEP_FRAMES=4
run SLB_LOCKSTEP_FRAMES=4 SLB_GROUP=14 SLB_CHUNK=28
run SLB_LOCKSTEP_FRAMES=3
run SLB_LOCKSTEP_FRAMES=1
run SLB_GROUP=49 SLB_CHUNK=49
run SLB_GROUP=25 SLB_CHUNK=50
run SLB_GROUP=17 SLB_CHUNK=51
run SLB_STREAMS=2
run SLB_STREAMS=3

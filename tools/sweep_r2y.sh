#!/bin/bash
# 2D 512^2 x 32 knob re-sweep after the 32x16 fused rows plan (device batch + e2e host batch)
cd "$(dirname "$0")/.."
run() { env "$@" python bench.py --no-3d --no-cpu-baseline --steps 40 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value']), round(d['e2e']['value']))"; }
run SLB_X=0
run SLB_STREAMS=4
run SLB_STREAMS=8
run SLB_GROUP=14
run SLB_GROUP=49 SLB_CHUNK=49
run SLB_LOCKSTEP_FRAMES=4
run SLB_LOCKSTEP_FRAMES=3
run SLB_GROUP2=7
run SLB_GROUP2=28
run SLB_HOST_PIPE=5
run SLB_X=0

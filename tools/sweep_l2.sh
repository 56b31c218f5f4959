#!/bin/bash
# 2D 512^2 device-batch schedule sweep: lock-step frame count x band chunk/group
cd "$(dirname "$0")/.."
run() { env "$@" python bench.py --no-3d --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value']), round(d['e2e']['value']), {k: round(v['ms_total']/v['bands']*1000,3) for k,v in d['kernels'].items() if v['bands']>100})"; }
run SLB_X=0
run SLB_LOCKSTEP_FRAMES=8 SLB_GROUP=4 SLB_CHUNK=4
run SLB_LOCKSTEP_FRAMES=8 SLB_GROUP=7 SLB_CHUNK=7
run SLB_LOCKSTEP_FRAMES=8 SLB_GROUP=2 SLB_CHUNK=2
run SLB_LOCKSTEP_FRAMES=4 SLB_GROUP=7 SLB_CHUNK=7
run SLB_LOCKSTEP_FRAMES=4 SLB_GROUP=4 SLB_CHUNK=4
run SLB_LOCKSTEP_FRAMES=2 SLB_GROUP=7 SLB_CHUNK=7
run SLB_LOCKSTEP_FRAMES=2 SLB_GROUP=14 SLB_CHUNK=14
run SLB_LOCKSTEP_FRAMES=8 SLB_GROUP=4 SLB_CHUNK=4 SLB_STREAMS=1

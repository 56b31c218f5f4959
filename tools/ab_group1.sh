#!/bin/bash
# e2e probe across the band group used inside the pipelined host batch (SLB_GROUP2; r1p measured it as SLB_GROUP1 before the split)
cd "$(dirname "$0")/.."
for r in 1 2; do for g in "" 4 10 14 25 49; do
  echo "[SLB_GROUP2=${g:-default}] $(env ${g:+SLB_GROUP2=$g} timeout 120 python tools/e2e_probe.py 8 2>&1 | head -1)"
done; done

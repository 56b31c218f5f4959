#!/bin/bash
# A/B of the pipelined host batch knobs (SLB_PIPE_GROUP, SLB_PIPE_CONC,
# SLB_HOST_PIPE, SLB_GROUP1) with the e2e probe, 2 rounds, 8 frames of 512^2
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in "" "SLB_PIPE_CONC=4" "SLB_PIPE_GROUP=2" "SLB_PIPE_GROUP=2 SLB_PIPE_CONC=4" \
           "SLB_PIPE_GROUP=2 SLB_HOST_PIPE=2" "SLB_PIPE_GROUP=2 SLB_HOST_PIPE=2 SLB_PIPE_CONC=4" \
           "SLB_PIPE_GROUP=2 SLB_HOST_PIPE=4 SLB_PIPE_CONC=4" "SLB_HOST_PIPE=4 SLB_PIPE_CONC=4"; do
    echo "[$v] $(env $v timeout 120 python tools/e2e_probe.py 8 2>&1 | head -1)"
  done
done

#!/bin/bash
# pipelined host batch schedules (e2e) at 8 and 32 frames of 512^2
cd "$(dirname "$0")/.."
for e in "SLB_X=0" "SLB_PIPE_HEAD=1 SLB_PIPE_GROUP=2" "SLB_PIPE_HEAD=2 SLB_PIPE_GROUP=2" "SLB_PIPE_HEAD=1 SLB_PIPE_GROUP=2 SLB_HOST_PIPE=4" "SLB_PIPE_HEAD=1 SLB_PIPE_GROUP=2 SLB_HOST_PIPE=4 SLB_PIPE_CONC=4" "SLB_PIPE_HEAD=2 SLB_PIPE_GROUP=2 SLB_HOST_PIPE=4 SLB_PIPE_CONC=4"; do
  echo "== $e"; env $e python tools/e2e_frames.py
done

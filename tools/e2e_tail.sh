#!/bin/bash
# pipelined host batch: the last SLB_PIPE_TAIL frames as singles (e2e at 16 / 32 frames)
cd "$(dirname "$0")/.."
for t in ${TAILS:-0 1 2 3 4 6 8}; do
  echo "== SLB_PIPE_TAIL=$t"; SLB_PIPE_TAIL=$t python tools/e2e_frames.py | grep -v '"frames": 8,'
done

#!/bin/bash
# TMA pipeline configuration sweep: consumer warps per CTA x ring stages (B=64, 10 it).
for w in 8 4; do for s in 2 3 4; do
  echo "== warps=$w stages=$s"
  QCL_PIPE_WARPS=$w QCL_PIPE_STAGES=$s timeout 60 python tools/engine_compare.py 10 64,128 0 2>&1 | grep "B="
done; done

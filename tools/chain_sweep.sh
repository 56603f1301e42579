#!/bin/bash
# Lane-group width x independent chains sweep (TMA engine, B=64 and 128, 10 iterations).
for cfg in "32 1" "32 2" "16 4" "16 2" "8 8" "8 4"; do
  set -- $cfg
  echo "== lanes=$1 chains=$2"
  QCL_LANES=$1 QCL_CHAINS=$2 timeout 60 python tools/engine_compare.py 10 64,128 0 2>&1 | grep "B="
done

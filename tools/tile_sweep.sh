#!/bin/bash
# Tile-size sweep of the TMA engine (items per consumer thread per tile) vs the direct engine.
for it in 1 2 4; do echo "== QCL_TILE_ITEMS=$it"; QCL_TILE_ITEMS=$it python tools/engine_compare.py 10 2>&1 | grep "B=64"; done

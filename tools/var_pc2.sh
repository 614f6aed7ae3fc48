#!/bin/bash
# PC2 sweep time per variant: tools/var_pc2.sh geom...
for v in paper_1709_01126_b200/variants/*.so; do
  echo "== $v"
  POT3D_LIB=$v timeout 300 python tools/sweep_geom.py "$@" 2>&1 | grep tiles
done

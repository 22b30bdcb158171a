#!/bin/bash
# A/B of lane-kernel variants (HS_LANE_VARIANT, see launch_batch in hs_kernels.cu)
for v in ${VARIANTS:-0 1 2 3}; do
  for d in "uniform naive" "normal8 adaptive" "normal32 adaptive" "normal64 adaptive" "const127 adaptive"; do
    echo -n "v=$v "; HS_LANE_VARIANT=$v python tools/kbench.py $d lane $((1<<30)) 10
  done
done

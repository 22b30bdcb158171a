#!/bin/bash
# tuning sweep of the lane-private kernel's batch size (U) and L2 prefetch distance (PF)
for cfg in "8 0" "8 1" "8 2" "6 0" "4 0" "4 2"; do
  set -- $cfg
  for d in "uniform naive" "normal32 adaptive" "const127 adaptive"; do
    echo -n "U=$1 PF=$2 "; HS_LANE_U=$1 HS_LANE_PF=$2 python tools/kbench.py $d lane $((1<<30)) 8
  done
done

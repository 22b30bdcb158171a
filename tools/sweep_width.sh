#!/bin/bash
# k_lane vs k_warp across distribution widths (1 GiB, device-resident)
for d in normal2 normal4 normal8 normal16 normal32 normal64 uniform const127; do
  python tools/kbench.py $d adaptive lane $((1<<30)) 8
  python tools/kbench.py $d naive warp $((1<<30)) 8
done

#!/bin/bash
# A/B of how a call's first launch orders itself behind its stream predecessor
# (HS_FIRST_LAUNCH 0/1/2 in hs_kernels.cu): back-to-back calls, CUDA events.
cd "$(dirname "$0")/../.."
for v in tools/ablib/first0.so paper_1011_0235_b200/_lib/libhist256.so tools/ablib/first2.so; do
  echo "== $v"; HS_LIBHIST256=$v python tools/diag/chained_ab.py
done

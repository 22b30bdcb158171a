#!/bin/bash
# same-box A/B of libhist256 builds in tools/ablib/ (kbench, interleaved rounds)
for round in 1 2; do
  for cfg in "lib_af55634 1024" "lib_cur 768" "lib_cur 769" "lib_cur 1025"; do
    set -- $cfg
    for d in "normal8 adaptive" "const127 adaptive" "uniform naive"; do
      echo -n "r$round $1 hot_threads=$2 "; HS_HOT_THREADS=$2 HS_LIBHIST256=tools/ablib/$1.so python tools/kbench.py $d lane $((1<<30)) 12 2>&1 | grep -v Warn
    done
  done
done

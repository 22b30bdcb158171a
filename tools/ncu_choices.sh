#!/bin/bash
# ncu counters for every kernel choice x distribution (kbench, 256 MiB, one launch each)
M=gpu__time_duration.sum,dram__bytes_read.sum.per_second,smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed
out=gpurun_out/ncu_choices.csv
: > $out
for d in uniform normal8 const127; do
  for ki in "naive warp" "adaptive subbin" "naive lane" "adaptive lane"; do
    python tools/kbench.py $d $ki $((256<<20)) 2 > /dev/null 2>&1 || { echo "plain run failed: $d $ki"; continue; }
    ncu --metrics $M --clock-control none -k regex:"k_(warp|subbin|lane)" -s 1 -c 1 --csv python tools/kbench.py $d $ki $((256<<20)) 2 2>/dev/null \
      | grep -E '^"[0-9]' | sed "s|^|\"$d\",\"$ki\",|" >> $out
  done
done
wc -l $out

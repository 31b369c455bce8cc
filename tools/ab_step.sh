#!/bin/bash
# A/B step time of two builds (build/ab/lib_base.so vs build/ab/lib_new.so, alternating, 3x each; GPU box):
#   bash tools/ab_step.sh <outdir under gpurun_out>
o=gpurun_out/${1:-ab}; mkdir -p $o
for i in 1 2 3; do
  for v in base new; do
    echo "$v $(RF_LIB_PATH=build/ab/lib_$v.so python tools/ablate_time.py | tail -1)" >> $o/ab.txt
  done
done
cat $o/ab.txt

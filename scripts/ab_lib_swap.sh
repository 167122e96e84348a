#!/bin/bash
# Same-box A/B of two builds of libzob200.so (file swap, no rebuild on the box):
#   gpurun -- 'bash scripts/ab_lib_swap.sh ab_old/libzob200_<rev>.so "<command>"'
set -u
OLD=${1:-ab_old/libzob200_e841f5c.so}
CMD=${2:-python scripts/bench_sampler.py}
mkdir -p gpurun_out
N=paper_2605_28760_b200/_build/libzob200.so
cp $N /tmp/new.so
for L in $OLD /tmp/new.so $OLD /tmp/new.so; do
  cp $L $N
  echo "== $L: $($CMD 2>&1 | tail -1)" >> gpurun_out/abl.txt
done
cp /tmp/new.so $N

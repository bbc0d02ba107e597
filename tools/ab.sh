#!/bin/bash
# A/B of two library builds inside one GPU session: alternating bench runs.
#   tools/ab.sh A.so B.so [rounds]
A=$1; B=$2; N=${3:-2}
for i in $(seq 1 $N); do
  for L in $A $B; do
    printf "%-24s " $(basename $L)
    ICB_LIB=$L python bench.py --steps 256 --warmup 16 --no-cpu-baseline 2>&1 | tail -1 | python tools/summ.py | cut -c1-90
  done
done

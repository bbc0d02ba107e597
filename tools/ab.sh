#!/bin/bash
# A/B of two library builds inside one GPU session: alternating bench runs.
#   tools/ab.sh A.so B.so [rounds] [extra bench args...]
A=$1; B=$2; N=${3:-2}; shift 3; EXTRA="$@"
for i in $(seq 1 $N); do
  for L in $A $B; do
    printf "%-28s " $(basename $L)
    ICB_LIB=$L python bench.py --steps 128 --warmup 8 --no-cpu-baseline $EXTRA 2>&1 | tail -1 | python tools/summ.py | cut -c1-110
  done
done

#!/bin/bash
# A/B of variant libraries on the GPU box: scripts/ab.sh "<lib list>" "<workload list>" "<precision list>"
for wl in ${2:-plaza_1m}; do
 for lib in $1; do
  for prec in ${3:-mixed f32}; do
    echo "== $lib $prec $wl"
    ORCA_B200_LIB=$PWD/variants/$lib.so python bench.py --resident-only --precision $prec --steps 100 --warmup 10 --workload $wl
  done
 done
done

#!/bin/bash
# A/B of variant libraries on the GPU box: scripts/ab.sh "<lib list>" "<extra bench args>"
for lib in $1; do
  for prec in mixed f32; do
    echo "== $lib $prec $2"
    ORCA_B200_LIB=$PWD/variants/$lib.so python bench.py --resident-only --precision $prec --steps 100 --warmup 10 $2
  done
done

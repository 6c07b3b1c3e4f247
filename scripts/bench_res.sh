#!/bin/bash
# resident-only bench over workloads x precisions with the in-tree library (or ORCA_B200_LIB)
for wl in ${1:-plaza_1m config3_262k_d1}; do
  for prec in ${2:-mixed f32}; do
    echo "== $wl $prec"
    python bench.py --resident-only --precision $prec --steps 100 --warmup 10 --workload $wl | cut -c1-400
  done
done

#!/bin/bash
# compact A/B of variant libraries on the GPU box: WL="<workloads>" PREC=<precision> scripts/ab2.sh <lib> ...
# (variants/<lib>.so, built with `make -C paper_2008_11578_b200/csrc OUT=$PWD/variants/<lib>.so EXTRA=-D...`)
for wl in ${WL:-plaza_1m}; do
for lib in "$@"; do
  for rep in 1 2; do
  ORCA_B200_LIB=$PWD/variants/$lib.so python bench.py --resident-only --steps 200 --warmup 10 --workload $wl ${PREC:+--precision $PREC} 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$wl', '$lib', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
  done
done
done

for lib in "$@"; do
  for rep in 1 2; do
  ORCA_B200_LIB=$PWD/variants/$lib.so python bench.py --resident-only --steps 200 --warmup 10 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
  done
done

for wl in plaza_1m config3_262k_d1 config3_262k_d2; do
 for sp in 0 1 0 1; do
  for prec in mixed f32; do
    echo "== spill=$sp $prec $wl"
    ORCA_FB_SPILL=$sp python bench.py --resident-only --precision $prec --steps 100 --warmup 10 --workload $wl
  done
 done
done

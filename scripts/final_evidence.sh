set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/g_mixed.json 2> gpurun_out/g_mixed.err
python bench.py --precision f32 > gpurun_out/g_f32.json 2>/dev/null
python bench.py --precision f64 > gpurun_out/g_f64.json 2>/dev/null
python bench.py --impl reference > gpurun_out/g_ref.json 2>/dev/null
rm -f gpurun_out/g_configs.jsonl
for wl in config1_1k config2_16k config3_262k_d1 config3_262k_d2 config5_8m; do python bench.py --workload $wl >> gpurun_out/g_configs.jsonl 2>/dev/null; done
ORCA_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 3 --warmup 3 --resident-only > gpurun_out/g_l.log 2>&1
ORCA_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:"k_solve_group|k_gather_fast32|k_scatter|k_fallback_coop|k_count|k_gather" -s 40 -c 7 -o gpurun_out/g_full python bench.py --steps 3 --warmup 4 --resident-only > gpurun_out/g_f.log 2>&1
ORCA_GRAPH=0 ncu --set full --clock-control none -k regex:"k_solve_group|k_fallback_coop" -s 12 -c 3 -o gpurun_out/g_full_d2 python bench.py --steps 3 --warmup 4 --resident-only --workload config3_262k_d2 > gpurun_out/g_fd2.log 2>&1
ls -la gpurun_out/g_*

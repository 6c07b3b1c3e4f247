# One gpurun call that produces everything profiles/ holds for the round (development tooling):
#   gpurun -- 'bash scripts/final_evidence.sh'    then    python scripts/refresh_profiles.py r02
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/g_default.json 2> gpurun_out/g_default.err
python bench.py --precision mixed --no-extras > gpurun_out/g_mixed.json 2>/dev/null
python bench.py --precision f32 --no-extras > gpurun_out/g_f32.json 2>/dev/null
python bench.py --precision f64 --no-extras > gpurun_out/g_f64.json 2>/dev/null
python bench.py --impl reference > gpurun_out/g_ref.json 2>/dev/null
rm -f gpurun_out/g_configs.jsonl gpurun_out/g_lp.jsonl gpurun_out/g_strips.jsonl
for wl in config1_1k config2_16k config3_262k_d1 config3_262k_d2 config3_262k_d1_nr3 config3_262k_d2_nr3 blobs_1m config5_8m; do python bench.py --workload $wl --no-extras >> gpurun_out/g_configs.jsonl 2>/dev/null; done
for wl in lp_1m_feasible lp_1m_half lp_1m_infeasible; do for p in f64 f32; do python bench.py --workload $wl --precision $p >> gpurun_out/g_lp.jsonl 2>/dev/null; done; done
# the multi-rank path on this one-GPU box: one rank over NCCL, then 2 and 4 ranks (processes) sharing the GPU --
# through peer-memory windows (CUDA IPC; the default transport) and through send/recv (gloo, staged through the host)
ORCA_BENCH_FORCE_STRIPS=1 python bench.py --steps 50 >> gpurun_out/g_strips.jsonl 2>/dev/null
python bench.py --gpus 2 --steps 30 >> gpurun_out/g_strips.jsonl 2>/dev/null
python bench.py --gpus 4 --steps 20 --workload config5_8m --scaling strong >> gpurun_out/g_strips.jsonl 2>/dev/null
python bench.py --gpus 2 --steps 30 --transport sendrecv >> gpurun_out/g_strips.jsonl 2>/dev/null
python bench.py --gpus 4 --steps 20 --workload config5_8m --scaling strong --transport sendrecv >> gpurun_out/g_strips.jsonl 2>/dev/null
ORCA_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 3 --warmup 3 --resident-only > gpurun_out/g_l.log 2>&1
# (--set full captures with ORCA_CHUNKS=1: one launch per kernel and step, the launches bench.py's per-stage timing and
#  roofline.traffic refer to; the launch list above shows the real step, two chunks)
ORCA_CHUNKS=1 ORCA_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:"k_solve_group|k_gather_fast32|k_scatter|k_fallback_coop|k_count|k_gather" -s 40 -c 7 -o gpurun_out/g_full python bench.py --steps 3 --warmup 4 --resident-only --precision mixed > gpurun_out/g_f.log 2>&1
ORCA_CHUNKS=1 ORCA_GRAPH=0 ncu --set full --clock-control none -k regex:"k_solve_group|k_fallback_coop" -s 12 -c 3 -o gpurun_out/g_full_d2 python bench.py --steps 3 --warmup 4 --resident-only --workload config3_262k_d2 --precision mixed > gpurun_out/g_fd2.log 2>&1
ORCA_CHUNKS=1 ORCA_GRAPH=0 ncu --set full --clock-control none -k regex:"k_solve_cert|k_solve_group_queue|k_shuffle" -s 6 -c 3 -o gpurun_out/g_full_cert python bench.py --steps 3 --warmup 4 --resident-only --precision cert32 > gpurun_out/g_fc.log 2>&1
ncu --set full --clock-control none -k regex:k_lp_batch -s 4 -c 2 -o gpurun_out/g_full_lp python bench.py --workload lp_1m_infeasible --steps 2 --warmup 3 > gpurun_out/g_flp.log 2>&1
# the reference's own test-suite against this package (tests/test_gpu_refsuite.py runs the same command)
PYTHONPATH=tests/refsuite:$PWD python -m pytest baseline/_ref/_tests -v -p no:cacheprovider > gpurun_out/g_refsuite.log 2>&1
# the reports are ~15 MB each and gpurun_out/ travels back only below 64 MiB: keep their raw pages instead
for f in g_full g_full_d2 g_full_cert g_full_lp; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null && rm -f gpurun_out/$f.ncu-rep; done
ls -la gpurun_out/g_*

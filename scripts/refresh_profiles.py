#!/usr/bin/env python
"""Turn one scripts/final_evidence.sh run (gpurun_out/g_*) into the tracked files under profiles/
(development tooling):   python scripts/refresh_profiles.py <tag>      e.g. tag = g"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"


def summary(kind, src):
    return subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), kind, src],
                          capture_output=True, text=True, check=True).stdout


def last_json_line(path):
    with open(path) as f:
        lines = [l for l in f.read().splitlines() if l.startswith("{")]
    return lines[-1]


# bench lines
for name in ("default", "mixed", "f32", "f64", "ref"):
    with open(os.path.join(P, f"bench_{tag}_{name}.json"), "w") as f:
        f.write(last_json_line(os.path.join(G, f"g_{name}.json")) + "\n")
for name in ("configs", "lp", "strips"):
    shutil.copy(os.path.join(G, f"g_{name}.jsonl"), os.path.join(P, f"bench_{tag}_{name}.jsonl"))

# the reference's own suite against this package: the verbose pytest listing as it came
rs = os.path.join(G, "g_refsuite.log")
if os.path.exists(rs):
    with open(rs) as f:
        lines = [l.rstrip() for l in f.read().splitlines()]
    keep = [l for l in lines if "::" in l or " passed" in l or " failed" in l or "error" in l.lower()]
    with open(os.path.join(P, f"{tag}_refsuite.txt"), "w") as f:
        f.write("# The reference's own test-suite (pkg/tests, unmodified, staged into baseline/_ref/_tests) with the name\n"
                "# `orcasim` bound to paper_2008_11578_b200 (tests/refsuite/orcasim), on one B200:\n"
                "#   PYTHONPATH=tests/refsuite:$PWD python -m pytest baseline/_ref/_tests -v -p no:cacheprovider\n\n")
        f.write("\n".join(keep) + "\n")

# ncu launch list and full captures
head_l = (f"# {tag} — ncu launch list of the default bench command (1,048,576 agents, `cert32`), final state of the round\n\n"
          "Command: `ORCA_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python "
          "bench.py --steps 3 --warmup 3 --resident-only` (per-launch times are cold-cache and serialised: compare "
          "shares; `k_import_*`, `k_iota`, `k_bbox`, `k_begin_bins`, `k_permute_rows` run once after the upload; the "
          "first `k_gather` launch searches for every agent, ~0.9 ms, the others ~25 us).\n\n")
with open(os.path.join(P, f"{tag}_launches_default_1m.md"), "w") as f:
    f.write(head_l + summary("launches", os.path.join(G, "g_launches.csv")))
head_f = (f"# {tag} — ncu --set full, kernels of the step, 1,048,576 agents, mixed precision, final state "
          "of the round\n\nCommand: `ORCA_GRAPH=0 ncu --set full --clock-control none --import-source on -k "
          "regex:\"k_solve_group|k_gather_fast32|k_scatter|k_fallback_coop|k_count|k_gather\" -s 40 -c 7 python "
          "bench.py --steps 3 --warmup 4 --resident-only`\n\n")
with open(os.path.join(P, f"{tag}_full_mixed_1m.md"), "w") as f:
    f.write(head_f + summary("full", os.path.join(G, "g_full.ncu-rep")))
head_d = (f"# {tag} — ncu --set full, solve and fallback kernels, 266,240 agents at 2.0 /m2 (79 % of the "
          "agents in the least-penetration stage), mixed precision\n\nCommand: `ORCA_GRAPH=0 ncu --set full "
          "--clock-control none -k regex:\"k_solve_group|k_fallback_coop\" -s 12 -c 3 python bench.py --steps 3 "
          "--warmup 4 --resident-only --workload config3_262k_d2`\n\n")
with open(os.path.join(P, f"{tag}_full_mixed_dense2.md"), "w") as f:
    f.write(head_d + summary("full", os.path.join(G, "g_full_d2.ncu-rep")))


with open(os.path.join(P, f"{tag}_full_cert32_1m.md"), "w") as f:
    f.write(f"# {tag} -- ncu --set full, the solve stage of ORCA_CERT32 (k_shuffle, k_solve_cert, k_solve_group_queue), "
            "1,048,576 agents\n\nCommand: `ORCA_GRAPH=0 ncu --set full --clock-control none -k "
            "regex:\"k_solve_cert|k_solve_group_queue|k_shuffle\" -s 6 -c 3 python bench.py --steps 3 --warmup 4 "
            "--resident-only --precision cert32`\n\n" + summary("full", os.path.join(G, "g_full_cert.ncu-rep")))
with open(os.path.join(P, f"{tag}_full_lp_infeasible.md"), "w") as f:
    f.write(f"# {tag} -- ncu --set full, batched LP (BASELINE config 4), 1,048,576 problems, infeasible mix, FP64\n\n"
            "Command: `ncu --set full --clock-control none -k regex:k_lp_batch -s 4 -c 2 python bench.py --workload "
            "lp_1m_infeasible --steps 2 --warmup 3`\n\n" + summary("full", os.path.join(G, "g_full_lp.ncu-rep")))

# traffic.json: DRAM bytes per launch and issue / pipe utilisation of the 1 M mixed capture
def raw_rows(rep):
    pre = rep[:-len(".ncu-rep")] + ".raw.csv" if rep.endswith(".ncu-rep") else rep
    if os.path.exists(pre):       # `ncu -i X.ncu-rep --page raw --csv > X.raw.csv` done on the GPU box (reports are big)
        out = open(pre).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def traffic_entry(rep, source):
    global col, units
    hdr, units, rows = raw_rows(rep)
    col = {k: i for i, k in enumerate(hdr)}
    entry = {"source": source, "ncu": {}}
    for r in rows:
        name = r[col["Kernel Name"]]
        short = name.split("<")[0].split()[-1].split("::")[-1]
        if short in entry:
            continue
        if short == "k_fallback_coop" and ", 16>" in name.split("(")[0]:
            continue          # the short-queue instance exits at once on this workload
        entry[short] = int(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"))
        entry["ncu"][short] = {
            "ipc": round(val(r, "sm__inst_executed.avg.per_cycle_elapsed"), 3),
            "fp64_pipe_pct": round(val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "lanes": round(val(r, "smsp__thread_inst_executed_per_inst_executed.ratio"), 2),
            "warps_pct": round(val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"), 1)}
    return entry


hdr, units, rows = raw_rows(os.path.join(G, "g_full.ncu-rep"))
col = {k: i for i, k in enumerate(hdr)}


def val(r, key):
    v = float(r[col[key]].replace(",", ""))
    u = units[col[key]]
    return v * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)


entry = {"source": f"profiles/{tag}_full_mixed_1m.md", "ncu": {}}
for r in rows:
    name = r[col["Kernel Name"]]
    short = name.split("<")[0].split()[-1].split("::")[-1]
    if short in entry and short != "k_fallback_coop":
        continue
    if short == "k_fallback_coop" and ", 16>" in name.split("(")[0]:
        continue          # the short-queue instance exits at once on this workload
    entry[short] = int(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"))
    entry["ncu"][short] = {
        "ipc": round(val(r, "sm__inst_executed.avg.per_cycle_elapsed"), 3),
        "fp64_pipe_pct": round(val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
        "lanes": round(val(r, "smsp__thread_inst_executed_per_inst_executed.ratio"), 2),
        "warps_pct": round(val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"), 1)}
tj = os.path.join(P, "traffic.json")
with open(tj) as f:
    t = json.load(f)
t["plaza_1m/mixed"] = entry
cert = traffic_entry(os.path.join(G, "g_full_cert.ncu-rep"), f"profiles/{tag}_full_cert32_1m.md")
for k in ("k_gather", "k_fallback_coop", "k_count", "k_scatter", "k_gather_fast32"):   # same kernels, same crowd
    cert.setdefault(k, entry.get(k))
    cert["ncu"].setdefault(k, entry["ncu"].get(k))
t["plaza_1m/cert32"] = cert
with open(tj, "w") as f:
    json.dump(t, f, indent=1)
    f.write("\n")
print(json.dumps(entry, indent=1))

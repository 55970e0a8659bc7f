"""Summarise a tools/gpu_evidence_r3.sh run (gpurun_out/ev_r3) into
profiles/r3/: bench lines, pytest / smoke / sanitizer results, the ncu
launch list of the driver's 20-step command, the --set full captures
(summary + hottest SASS lines), a SASS excerpt of the timed kernel, and
profiles/traffic.json (dram bytes per launch of the dominant kernels)."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "ev_r3")
# (SL_EVIDENCE_DST / SL_TRAFFIC_JSON: summarise on the GPU box itself, into
# gpurun_out/, when the raw ncu reports are too large to bring back)
DST = os.environ.get("SL_EVIDENCE_DST") or os.path.join(ROOT, "profiles", "r3")
os.makedirs(DST, exist_ok=True)

# bench lines
lines = {}
for f in sorted(os.listdir(SRC)):
    if f.startswith("bench_") and f.endswith(".json"):
        rows = [x for x in open(os.path.join(SRC, f)) if x.startswith("{")]
        if rows:
            lines[f[6:-5]] = json.loads(rows[-1])
with open(os.path.join(DST, "bench_lines.json"), "w") as fh:
    json.dump(lines, fh, indent=1)
for f in ("pytest.txt", "smoke.txt", "sanitizer.txt", "e2e_settle_B.txt",
          "e2e_settle_D.txt", "predicate.txt", "edit_latency.txt",
          "edit_latency_full.txt", "build_timing.txt", "e2e_trace_B20.txt"):
    if os.path.exists(os.path.join(SRC, f)):
        shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))

# launch list of the driver's command (20 timed steps)
p = os.path.join(SRC, "launches_n20.csv")
if os.path.exists(p):
    raw = open(p).read().splitlines()
    start = [i for i, l in enumerate(raw) if l.startswith('"ID"')][0]
    rows = list(csv.reader(raw[start:]))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    with open(os.path.join(DST, "launches_n20.txt"), "w") as out:
        out.write("# ncu --metrics gpu__time_duration.sum --clock-control "
                  "none: python bench.py --steps 20 --warmup 5 --no-e2e "
                  "--no-cpu-baseline --no-fp64\n# (cold-cache, serialised "
                  "launches: compare shares, not absolute times)\n")
        for r in rows[1:]:
            name = r[ik].split("(")[0].replace("void ", "")
            ns = float(r[iv])
            t = tot.setdefault(name, [0, 0.0])
            t[0] += 1
            t[1] += ns
            out.write(f"{name:52s} {ns / 1000:9.2f} us\n")
        out.write("\n# totals\n")
        allt = sum(v[1] for v in tot.values())
        for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
            out.write(f"{k[:60]:60s} n={v[0]:4d} {v[1] / 1000:10.2f} us  "
                      f"share {100 * v[1] / allt:5.1f}%\n")

# --set full captures: (report, algorithmic bytes per launch)
algo = {"win_fp32": lines.get("default", {}).get("roofline", {}).get(
            "algorithmic_bytes_per_step"),
        "win_fp64": 409563104, "win_mixed": 307708736,
        "fused": None, "split_atomic": None, "mass": None,
        "win_E200": lines.get("E1", {}).get("roofline", {}).get(
            "algorithmic_bytes_per_step_per_gpu")}
traffic = {"_source": "ncu --set full (profiles/r3/ncu_*.txt): "
                      "dram__bytes_read.sum + dram__bytes_write.sum of one "
                      "launch of the dominant kernel per workload"}
keys = {"win_fp32": "100^3/fp32/gather", "win_fp64": "100^3/fp64/gather",
        "win_mixed": "100^3/mixed/gather", "win_E200": "E200/fp32/gather"}
for name, ab in algo.items():
    rep = os.path.join(SRC, f"prof_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = os.path.join(DST, f"ncu_{name}.txt")
    args = [sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
            rep, out] + ([str(int(ab))] if ab else [])
    subprocess.run(args, check=True, stdout=subprocess.DEVNULL)
    with open("/tmp/_src.csv", "w") as fh:
        subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                        "--print-source", "sass"], stdout=fh,
                       stderr=subprocess.DEVNULL)
    with open(os.path.join(DST, f"ncu_{name}_hot.txt"), "w") as fh:
        subprocess.run([sys.executable,
                        os.path.join(ROOT, "tools", "ncu_hot.py"),
                        "/tmp/_src.csv", "25"], stdout=fh)
    for l in open(out):
        if l.startswith("traffic (dram r+w) bytes") and name in keys:
            traffic[keys[name]] = int(float(l.split()[-1]))
with open(os.environ.get("SL_TRAFFIC_JSON") or
          os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)

# SASS of the timed kernel: the TMA / mbarrier / elect instructions
obj = os.path.join(ROOT, "paper_1911_10274_b200", "build",
                   "sl_kernels_fp32.o")
fn = "_ZN2sl9k_win_tmaILi1ELi16EEEvNS_6KStateENS_4EnvPENS_5StepPENS_6WinCfgE"
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj],
                      capture_output=True, text=True).stdout.splitlines()
keep = [l.strip() for l in sass if any(k in l for k in (
    "UBLKCP", "SYNCS", "ELECT", "MUFU.RSQ", "FADD2", "ACQBULK",
    "UTMALDG", "griddep", "ACQ", "CCTL"))]
with open(os.path.join(DST, "sass_k_win_tma_fp32_T16.txt"), "w") as fh:
    fh.write(f"# cuobjdump -sass -fun {fn} {os.path.relpath(obj, ROOT)}\n"
             f"# {len(sass)} lines; the bulk-copy (UBLKCP), mbarrier "
             f"(SYNCS), elect, packed fp32x2 and MUFU.RSQ instructions:\n")
    fh.write("\n".join(keep) + "\n")
print("saved to", DST)

"""Copy one gpu_evidence.sh run (gpurun_out/*_TAG*) into profiles/: bench
lines, pytest summary, the ncu launch list (summarised) and the --set full
capture summary + hottest SASS lines of the dominant kernel.
usage: python tools/save_evidence.py TAG [algorithmic_bytes]"""
import csv
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
algo = sys.argv[2] if len(sys.argv) > 2 else "255708736"
src, dst = "gpurun_out", "profiles"
for f in os.listdir(src):
    if tag in f and (f.endswith(".json") or f.startswith("pytest_")
                     or f.startswith("smoke_")):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
# launch list
lines = open(os.path.join(src, f"launches_{tag}.csv")).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = {}
with open(os.path.join(dst, f"launches_{tag}.txt"), "w") as out:
    out.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 60"
              ": python bench.py --steps 10 --warmup 3 --no-e2e "
              "--no-cpu-baseline\n# (cold-cache, serialised launches; compare "
              "shares, not absolutes)\n")
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "")
        ns = float(r[iv])
        t = tot.setdefault(name, [0, 0.0])
        t[0] += 1
        t[1] += ns
        out.write(f"{name:50s} {ns / 1000:9.2f} us\n")
    out.write("\n# totals\n")
    allt = sum(v[1] for v in tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
        out.write(f"{k[:60]:60s} n={v[0]:3d} {v[1] / 1000:10.2f} us  "
                  f"share {100 * v[1] / allt:5.1f}%\n")
rep = os.path.join(src, f"prof_{tag}.ncu-rep")
if os.path.exists(rep):
    subprocess.run([sys.executable, "tools/ncu_summary.py", rep,
                    os.path.join(dst, f"ncu_k_win_tma_fp32_{tag}.txt"), algo],
                   check=True, stdout=subprocess.DEVNULL)
    with open("/tmp/_src.csv", "w") as fh:
        subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                        "--print-source", "sass"], stdout=fh,
                       stderr=subprocess.DEVNULL)
    with open(os.path.join(dst, f"ncu_k_win_tma_fp32_{tag}_hot.txt"),
              "w") as fh:
        subprocess.run([sys.executable, "tools/ncu_hot.py", "/tmp/_src.csv",
                        "25"], stdout=fh)
# the other modes' window kernels and the fused small-body kernel
for name, out_name, ab in (("fp64", "ncu_k_win_tma_fp64", "409600000"),
                           ("mixed", "ncu_k_win_tma_mixed", "307700000"),
                           ("fused", "ncu_k_fused_small_fp32", "128400000")):
    rep = os.path.join(src, f"prof_{name}_{tag}.ncu-rep")
    if os.path.exists(rep):
        subprocess.run([sys.executable, "tools/ncu_summary.py", rep,
                        os.path.join(dst, f"{out_name}_{tag}.txt"), ab],
                       check=True, stdout=subprocess.DEVNULL)
print("saved", tag)

"""Lattice build + first device sync timings: the
host builder (sl_build_lattice on all host threads, bit-identical to the
numpy builder), the first push (uploads) and the device layout build, for
the 100^3 and 200^3 lattices."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig, engine  # noqa: E402

for n in (100, 200):
    t0 = time.perf_counter()
    st, env = bench.build_workload(n)
    t1 = time.perf_counter()
    cfg = StepConfig(dt=1e-4, precision="fp32")
    mir = engine.mirror_for(st, cfg)
    mir.push(st, env)
    mir.ctx.sync()
    t2 = time.perf_counter()
    mir.ctx.step([0.0], 1e-4, cfg.native_accumulation, mir.counters)
    mir.ctx.sync()
    t3 = time.perf_counter()
    print(f"{n}^3: {st.mass_count} masses, {st.spring_count} springs: "
          f"host build {1e3 * (t1 - t0):.0f} ms, upload {1e3 * (t2 - t1):.0f} "
          f"ms, device layout build + first step {1e3 * (t3 - t2):.0f} ms")
    engine.drop_mirrors(st)
    del st

import sys; sys.path[:0] = ["tests", "oracle", "."]
import numpy as np
from conftest import load_golden, case_context, case_times
g = load_golden(sys.argv[1] if len(sys.argv) > 1 else "cube10_contact")
ctx = case_context(g, "fp64")
c = np.zeros(3, np.int64)
ctx.step(case_times(g)[:3], float(g["dt"]), 0, c)
print("path", ctx.stats()["step_path"])

"""Q11 at p = 1..3 on 8^3 / 16^3 / 32^3 with the test's solver
(tests/test_oracle_pins.py::_solve_manufactured): the full-size record the CPU test
suite cannot afford at p = 3.  Output: one JSON line per degree."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cutgen  # noqa: E402
from test_oracle_pins import _solve_manufactured  # noqa: E402

cutgen.build()
for p in [int(a) for a in (sys.argv[1:] or ["1", "2", "3"])]:
    t0 = time.time()
    errs = [_solve_manufactured(cutgen, N, p) for N in (8, 16, 32)]
    eoc = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    print(json.dumps({"p": p, "meshes": [8, 16, 32], "l2_rel_err": errs, "eoc": eoc,
                      "bound": p + 0.7, "ok": min(eoc) >= p + 0.7, "seconds": round(time.time() - t0, 1)}),
          flush=True)

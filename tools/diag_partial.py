"""Print pivots / signed dets / swap flags of the device partial-pivoting run
on a partial golden case (debug aid for tests/test_partial_pivot.py)."""
import sys, os
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from test_partial_pivot import load_partial
from paper_1308_1536_b200.elim import eliminate
from paper_1308_1536_b200 import engine

name = sys.argv[1] if len(sys.argv) > 1 else "pp_int7_s0"
meta, A = load_partial(name)
orig = engine.DeviceElimination.swaps
got = {}
def spy(self, upto):
    r = orig(self, upto)
    got["sw"] = r
    return r
engine.DeviceElimination.swaps = spy
tr, _ = eliminate(A, collect_minors=False, pivot_mode="partial")
print("swaps", [int(x) for x in got["sw"]])
print("pivots", [float(x) for x in tr.pivots])
print("dets", [float(x) for x in tr.det_series])
print("final", [[float(x) for x in r] for r in A.rows])

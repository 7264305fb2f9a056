"""Debug helper: one small elimination vs the oracle (n, p, steps from argv)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import oracle  # noqa: E402
from _util import first_mismatch  # noqa: E402
from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

n, p, steps = map(int, sys.argv[1:4])
A = random_uniform_soa(n, p, seed=n + p)
ref = oracle.OracleRank(n, p, "real")
ref.load(A)
res_o = HostResults.alloc(n, 1, ref.L, True)
ref.run(True, True, 0, steps, res_o)
fin_o = A.copy()
ref.fetch(fin_o)
with DeviceElimination(n, p, "real") as eng:
    eng.load(A)
    res_d = HostResults.alloc(n, 1, eng.L, True)
    eng.run(True, True, 0, steps, res_d)
    fin_d = A.copy()
    eng.fetch(fin_d)
    print("counters", eng.counters())
print("mismatches:", first_mismatch(fin_o, fin_d, p))

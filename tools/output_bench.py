"""Time the result-file writers on one run's results (oracle results, CPU only).

usage: python tools/output_bench.py N P
native = write_results (csrc/hostio.c, all host threads); python = the CLI's
loops over scalar objects (output.write_dets / write_minors, what the
reference's cli._write_* do) including building the MinorRow objects."""
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import oracle  # noqa: E402

from paper_1308_1536_b200.elim import EliminationTrace, MinorSeries, minor_rows_from_results  # noqa: E402
from paper_1308_1536_b200.engine import HostResults  # noqa: E402
from paper_1308_1536_b200.output import write_dets, write_minors, write_results  # noqa: E402
from paper_1308_1536_b200.scalars import Precision  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

n, p = int(sys.argv[1]), int(sys.argv[2])
A = random_uniform_soa(n, p, 3)
ref = oracle.OracleRank(n, p, "real")
ref.load(A)
res = HostResults.alloc(n, 1, ref.L, True)
rc, done = ref.run(True, True, 0, n, res)
scalars = done + n * (n + 1) - 2  # dets + signed and normalized entries of sizes 2..n
with tempfile.TemporaryDirectory() as d1, tempfile.TemporaryDirectory() as d2:
    t0 = time.perf_counter()
    write_results(res, n, p, "real", d1, done)
    t1 = time.perf_counter()
    prec = Precision(p)
    trace = EliminationTrace(n=n, prec=prec)
    trace.det_series = [res.dets.get(i, p) for i in range(done)]
    minors = MinorSeries(prec)
    for row in minor_rows_from_results(res, n, p):
        minors.rows[row.n] = row
    write_dets(trace, os.path.join(d2, "dets.txt"), prec.decimal_digits)
    write_minors(minors, d2, prec.decimal_digits)
    t2 = time.perf_counter()
    same = all(open(os.path.join(d1, f), "rb").read() == open(os.path.join(d2, f), "rb").read()
               for f in os.listdir(d1))
print(f"N={n} p={p}: {scalars} scalars; native {t1 - t0:.3f}s on {len(os.sched_getaffinity(0))} threads, "
      f"python {t2 - t1:.3f}s ({(t2 - t1) / (t1 - t0):.0f}x); identical={same}")

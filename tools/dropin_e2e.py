"""End-to-end time of the DROP-IN call at benchmark size: paper_1308_1536_b200.
eliminate(A) on a MatrixBuffer (the reference's signature, elim.py:158), with
every MinorRow handed to the caller as scalar objects (sink / MinorSeries) and
A left as the in-place L\\U state -- i.e. what a user of the reference gets,
including the boundary conversions the C-ABI bench line does not pay.

usage: python tools/dropin_e2e.py [N] [BITS]     (default 2000 4096, random_uniform)
Prints one JSON line: seconds for eliminate(), of which the device run, the
scalar conversion of the minors rows, and the first materialisation of A."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1308_1536_b200 import MatrixBuffer, Precision, eliminate  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    soa = random_uniform_soa(n, p, seed=n)
    A = MatrixBuffer.from_soa(n, "real", Precision(p), soa)  # lazily materialised, like a loaded matrix
    torch.cuda.synchronize()
    rows = []
    t0 = time.perf_counter()
    trace, minors = eliminate(A, sink=rows.append)
    t1 = time.perf_counter()
    first = A.rows[n - 1][n - 1]  # materialise the in-place buffer (n^2 scalar objects)
    t2 = time.perf_counter()
    scalars = sum(len(r.signed) + (len(r.normalized) if r.normalized else 0) for r in rows)
    L = (p + 31) // 32
    work = n * (n - 1) ** 2 / 2 * L * L
    print(json.dumps({"n": n, "prec_bits": p, "eliminate_s": t1 - t0, "limb_mac_per_s": work / (t1 - t0),
                      "minor_rows": len(rows), "minor_scalars": scalars, "materialise_A_s": t2 - t1,
                      "det_n_exponent": int(trace.det_series[-1].as_mantissa_exp()[1]) if trace.det_series else None,
                      "note": "eliminate() streams rows from the device in chunks on a worker thread while this "
                              "thread converts them; A is materialised lazily (here: forced, timed separately)"}))


if __name__ == "__main__":
    main()

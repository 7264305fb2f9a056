"""Shared test helpers: golden fixtures, digests of SoA results."""
import glob
import json
import os

import numpy as np

from golden.digest import digest_parts
from paper_1308_1536_b200 import genmat, mp
from paper_1308_1536_b200.scalars import Precision
from paper_1308_1536_b200.soa import SoA

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ZEROS = os.path.join(os.path.dirname(GOLDEN), "..", "data", "zeta_zeros.txt")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    return meta, arrays


def build_input(meta, arrays) -> SoA:
    """Input matrix SoA: stored arrays, else regenerated with the product's
    builders (whose output the tests pin by fingerprint)."""
    if "in_limbs" in arrays:
        return SoA(arrays["in_limbs"].shape[0], arrays["in_limbs"].shape[1], arrays["in_limbs"].shape[2],
                   np.ascontiguousarray(arrays["in_limbs"]), np.ascontiguousarray(arrays["in_exp"]),
                   np.ascontiguousarray(arrays["in_cls"]))
    return generate(meta["gen"]).to_soa()


def generate(gen):
    fam = gen[0]
    if fam in ("random_uniform", "hilbert", "random_illcond"):
        return genmat.synth_matrix(fam, gen[1], gen[2], Precision(gen[3]))
    if fam == "beta":
        z = genmat.load_zeros(ZEROS, Precision(gen[2]), gen[1])
        return genmat.beta_matrix(z, gen[1], genmat.SpougeGamma(), Precision(gen[2]))
    if fam == "power":
        z = genmat.load_zeros(ZEROS, Precision(2048), gen[1])
        with mp.context(precision=2048):
            t = mp.mpfr(gen[2])
        return genmat.power_matrix(z, gen[1], t, Precision(gen[3]))
    raise ValueError(fam)


def results_digest(res, final: SoA, n: int, prec: int, done: int):
    piv = [res.pivots.canonical(i, prec) for i in range(done)]
    dets = [res.dets.canonical(i, prec) for i in range(done)]
    rows = []
    if res.signed is not None:
        for m in range(2, n + 1):
            fl = int(res.row_flags[m - 1])
            if not fl & 1:
                continue
            base = (m - 1) * n
            signed = [res.signed.canonical(base + k, prec) for k in range(m)]
            normalized = [res.normalized.canonical(base + k, prec) for k in range(m)] if fl & 2 else None
            rows.append((m, signed, normalized))
    fin = [final.canonical(i, prec) for i in range(final.count)]
    return digest_parts(piv, dets, rows, fin)


def first_mismatch(a: SoA, b: SoA, prec: int, limit=5):
    out = []
    for i in range(a.count):
        if a.canonical(i, prec) != b.canonical(i, prec):
            out.append((i, a.canonical(i, prec), b.canonical(i, prec)))
            if len(out) >= limit:
                break
    return out

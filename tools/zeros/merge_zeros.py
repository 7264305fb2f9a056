"""Merge gen_zeros.py outputs into a zeros file in the reference's format
(genmat.load_zeros / save_zeros; reference scripts/make_zeros.py:48-54).

usage: python merge_zeros.py BITS OUTFILE RAWFILE...
"""
import glob
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1308_1536_b200 import mp  # noqa: E402
from paper_1308_1536_b200.genmat import ZetaZeros, save_zeros  # noqa: E402

bits, out = int(sys.argv[1]), sys.argv[2]
raw = {}
for pat in sys.argv[3:]:
    for path in glob.glob(pat):
        for line in open(path):
            k, v = line.split()
            raw[int(k)] = v
count = max(raw)
missing = [k for k in range(1, count + 1) if k not in raw]
if missing:
    count = missing[0] - 1
with mp.context(precision=bits):
    gammas = [mp.mpfr(raw[k]) for k in range(1, count + 1)]
assert all(b > a for a, b in zip(gammas, gammas[1:]))
save_zeros(ZetaZeros(gammas, bits), out,
           f"first {count} nontrivial zeta zero ordinates\n"
           f"source precision: {bits} bits (mpmath zetazero, mp.prec = {bits + 64})\n"
           f"generated with tools/zeros/gen_zeros.py + merge_zeros.py")
print(f"wrote {count} zeros to {out}")

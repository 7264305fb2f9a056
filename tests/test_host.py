"""Host-side logic of the drop-in: scalars, SoA format, MatrixBuffer, wire
format, topology, and the generic (Fraction) primitives."""
import random
from fractions import Fraction

import numpy as np
import pytest

from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.elim import apply_pivot_to_row, minors_row_from_l, normalize_minors
from paper_1308_1536_b200.errors import CorruptPayload, NormalizationUndefined, PrecisionMismatch
from paper_1308_1536_b200.genmat import synth_matrix
from paper_1308_1536_b200.matrix import MatrixBuffer
from paper_1308_1536_b200.parexec import (WorkerTopology, block_reassign_plan, is_abort, pack_abort, pack_row,
                                          unpack_abort, unpack_row)
from paper_1308_1536_b200.scalars import (Precision, agree_digits, canonical_bits, format_scalar, parse_scalar,
                                          same_bits)
from paper_1308_1536_b200.soa import SoA


def test_precision_floor():
    with pytest.raises(ValueError):
        Precision(63)
    assert Precision(4096).limbs == 128 and Precision(33220).limbs == 1039


@pytest.mark.parametrize("bits", [64, 100, 256, 333, 4096])
def test_parse_format_round_trip(bits):
    prec = Precision(bits)
    A = synth_matrix("random_uniform", 4, bits, prec)
    for x in (v for row in A.rows for v in row):
        assert same_bits(parse_scalar(format_scalar(x), prec), x)
    with prec.context():
        z = -mp.mpfr(0)
    assert format_scalar(z) == "-0" and canonical_bits(z) == ("r", "-0")


@pytest.mark.parametrize("bits,kind", [(64, "real"), (65, "real"), (192, "complex"), (1000, "real"), (4097, "complex")])
def test_soa_round_trip(bits, kind):
    prec = Precision(bits)
    rs = mp.random_state(bits)
    with prec.context():
        vals = [2 * mp.mpfr_random(rs) - 1 for _ in range(20)] + [mp.mpfr(0), -mp.mpfr(0), mp.mpfr(2) ** 1000]
        if kind == "complex":
            vals = [mp.mpc(v, -v * 3) for v in vals]
    s = SoA.from_scalars(vals, bits, kind)
    assert s.limbs.shape == (2 if kind == "complex" else 1, (bits + 31) // 32, len(vals))
    for i, v in enumerate(vals):
        assert s.canonical(i, bits) == canonical_bits(v)
        assert same_bits(s.get(i, bits), v)
    # left-aligned: MSB set on every nonzero
    nz = s.cls == 0
    assert np.all((s.limbs[:, -1, :][nz | (s.cls == 1)] >> 31) == 1)


def test_matrix_soa_round_trip_and_fingerprint():
    A = synth_matrix("random_uniform", 7, 1, Precision(320))
    B = MatrixBuffer.from_soa(7, "real", Precision(320), A.to_soa())
    assert B.same_bits(A) and B.fingerprint() == A.fingerprint()


def test_precision_mismatch():
    with Precision(128).context():
        rows = [[mp.mpfr(1), mp.mpfr(2)], [mp.mpfr(3), mp.mpfr(4)]]
    with pytest.raises(PrecisionMismatch):
        MatrixBuffer(2, "real", Precision(256), rows)


def test_mpmat_round_trip(tmp_path):
    A = synth_matrix("random_uniform", 5, 2, Precision(200))
    A.save(tmp_path / "a.mpmat")
    assert MatrixBuffer.load(tmp_path / "a.mpmat").same_bits(A)


def test_exact_series_with_fraction_arithmetic():
    """The shared primitives run over exact rationals reproduce the cofactors
    exactly (the reference's test_elim.py:74-93 property)."""
    entries = [[Fraction(v) for v in r] for r in [[2, 1, 1, 3], [1, 3, 2, 1], [1, 0, 1, 2], [4, 1, 1, 1]]]
    rows = [list(r) for r in entries]
    det, dets = None, []
    for i in range(4):
        det = rows[i][i] if det is None else det * rows[i][i]
        dets.append(det)
        for j in range(i + 1, 4):
            apply_pivot_to_row(rows[j], rows[i], i)
        if i + 2 <= 4:
            m = i + 2
            signed = minors_row_from_l(rows[m - 1][:m - 1], dets[i])
            # cofactors of column m of the leading m x m block
            for k in range(m):
                sub = [[entries[r][c] for c in range(m - 1)] for r in range(m) if r != k]
                assert signed[k] == (-1) ** (k + m - 1) * _det(sub)


def _det(M):
    if not M:
        return Fraction(1)
    return sum((-1) ** j * M[0][j] * _det([r[:j] + r[j + 1:] for r in M[1:]]) for j in range(len(M)))


def test_normalize_minors():
    with Precision(256).context():
        out = normalize_minors([mp.mpfr(3), mp.mpfr(7), mp.mpfr(-2)])
        assert out[0] == 1 and agree_digits(out[1], mp.mpfr(7) / 3) > 70
        with pytest.raises(NormalizationUndefined):
            normalize_minors([mp.mpfr(0), mp.mpfr(1)])


def test_wire_round_trip_and_corruption():
    prec = Precision(128)
    rs = mp.random_state(4)
    with prec.context():
        xs = [2 * mp.mpfr_random(rs) - 1 for _ in range(4)] + [mp.mpfr(0), -mp.mpfr(0)]
    wire = pack_row(3, xs, "real")
    step, back = unpack_row(wire, prec, "real")
    assert step == 3 and all(same_bits(a, b) for a, b in zip(xs, back))
    rng = random.Random(0)
    for _ in range(40):
        w = bytearray(wire)
        w[rng.randrange(len(w))] ^= 1 << rng.randrange(8)
        with pytest.raises(CorruptPayload):
            unpack_row(bytes(w), prec, "real")
    assert is_abort(pack_abort(9, 2)) and unpack_abort(pack_abort(9, 2)) == (9, 2)


def test_topology_and_plan():
    t = WorkerTopology(3, 10)
    assert [t.owner(r) for r in range(1, 7)] == [1, 2, 3, 1, 2, 3] and t.owned_rows(2) == [2, 5, 8]
    for w in (1, 2, 3, 4, 7):
        sizes = [len(WorkerTopology(w, 23).owned_rows(k)) for k in range(1, w + 1)]
        assert max(sizes) - min(sizes) <= 1 and sum(sizes) == 23
    assert [last - first + 1 for _, first, last in block_reassign_plan(0, 10, 3)] == [4, 3, 3]
    with pytest.raises(ValueError):
        WorkerTopology(0, 5)


@pytest.mark.parametrize("p", [64, 65, 100, 1024, 1055])
def test_counter_uniform_is_exactly_2u_minus_1(p):
    """synth.counter_uniform_soa (host twin of the device builder): every element equals
    (k - 2^(p-1)) 2^(1-p) for the generator's p-bit integer k (genmat.py:242-246: 2U - 1 at p
    bits is exact), recomputed here with Python integers."""
    from fractions import Fraction
    import numpy as np
    from paper_1308_1536_b200.synth import counter_uniform_soa
    n, seed = 5, 11 + p
    L = (p + 31) // 32
    s = counter_uniform_soa(n, p, seed)
    M64 = 2 ** 64 - 1

    def mix(x):
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
        return x ^ (x >> 31)

    key = mix(seed ^ 0x243F6A8885A308D3)
    npairs = (L + 1) // 2
    for idx in range(n * n):
        K = 0
        for q in range(npairs):
            K |= mix((key + (idx * npairs + q + 1) * 0x9E3779B97F4A7C15) & M64) << (64 * q)
        K &= (1 << (32 * L)) - 1
        K &= ~((1 << (32 * L - p)) - 1)
        want = Fraction(K - 2 ** (32 * L - 1), 2 ** (32 * L - 1))
        got = s.get(idx, p)
        assert got._fraction() == want, idx


def test_scalars_pickle_and_copy():
    """Result scalars behave like gmpy2's: immutable (copy returns the object) and
    picklable bit-exactly -- including the pooled ones the boundary conversion makes."""
    import copy
    import pickle
    from paper_1308_1536_b200 import mp
    from paper_1308_1536_b200.scalars import canonical_bits
    from paper_1308_1536_b200.synth import random_uniform_soa
    s = random_uniform_soa(3, 333, seed=1)
    xs = s.scalars(0, 9, 333)
    for x in xs + [mp.mpfr(0), -mp.mpfr(0), mp.mpfr(1.5)]:
        y = pickle.loads(pickle.dumps(x))
        assert canonical_bits(y) == canonical_bits(x) and y.precision == x.precision
    c = mp.mpc_from_parts(xs[0], xs[1])
    assert canonical_bits(pickle.loads(pickle.dumps(c))) == canonical_bits(c)
    assert copy.copy(xs[0]) is xs[0] and copy.deepcopy([xs[2]])[0] is xs[2]

"""Result digests shared by the golden generator (reference objects) and the
tests (device / oracle SoA results).  Pure Python, no dependencies.

A digest is sha256 over repr() of canonical scalar forms -- the reference's
canonical_bits (scalars.py:129-145): ('r', odd mantissa, exponent) or
('r', '+0'/'-0'), complex ('c', re, im) -- in a fixed order:
pivots, det_series, then for each emitted size m: signed[0..m), normalized
or None, then the final matrix row-major."""

import hashlib


def digest_parts(pivots, dets, minor_rows, final_rows):
    h = hashlib.sha256()
    h.update(b"pivots")
    for x in pivots:
        h.update(repr(x).encode())
    h.update(b"dets")
    for x in dets:
        h.update(repr(x).encode())
    h.update(b"minors")
    for m, signed, normalized in minor_rows:
        h.update(f"m{m}".encode())
        for x in signed:
            h.update(repr(x).encode())
        if normalized is None:
            h.update(b"None")
        else:
            for x in normalized:
                h.update(repr(x).encode())
    h.update(b"final")
    for x in final_rows:
        h.update(repr(x).encode())
    return h.hexdigest()

"""Host multiprecision scalars with the gmpy2 API, over the system MPFR 4.2.1 /
MPC 1.3.1 / GMP 6.3.0 runtime libraries (ctypes; the headers are absent).

The reference keeps every matrix entry as a gmpy2.mpfr / gmpy2.mpc object
(scalars.py:1-12) and gmpy2 cannot be installed in this image.  This module
provides the same scalar objects for the drop-in's HOST side only:

* the matrix-family builders (genmat.py) -- input generation, reproduced op
  for op so inputs are bit-identical to the reference's;
* parse_scalar / format_scalar / MPMAT I/O (scalars.py, matrix.py);
* the user-visible scalars in EliminationTrace / MinorSeries / MatrixBuffer.

The elimination itself (eliminate / par_eliminate) never computes with these
objects: it packs them into the ds SoA format and runs on the B200 through
libdetseries_b200.so, and fails loudly when that library is missing.

Every arithmetic result is the correctly rounded (RNDN) MPFR/MPC result at
the active context precision, exactly like gmpy2; int/float operands are
converted exactly first.
"""

from __future__ import annotations

import ctypes
import math
import threading
from ctypes import (POINTER, Structure, byref, c_char_p, c_double, c_int, c_long,
                    c_size_t, c_ulong, c_void_p)
from fractions import Fraction

_LIB = "/usr/lib/x86_64-linux-gnu/"
_gmp = ctypes.CDLL(_LIB + "libgmp.so.10")
_mpfr = ctypes.CDLL(_LIB + "libmpfr.so.6")
_mpc = ctypes.CDLL(_LIB + "libmpc.so.3")

version = lambda: "2.1.5-shim"  # noqa: E731


class _MPFR_T(Structure):
    _fields_ = [("prec", c_long), ("sign", c_int), ("exp", c_long), ("d", POINTER(c_ulong))]


class _MPC_T(Structure):
    _fields_ = [("re", _MPFR_T), ("im", _MPFR_T)]


class _MPZ_T(Structure):
    _fields_ = [("alloc", c_int), ("size", c_int), ("d", POINTER(c_ulong))]


_PF = POINTER(_MPFR_T)
_PC = POINTER(_MPC_T)
_PZ = POINTER(_MPZ_T)

_EXP_ZERO = -0x7fffffffffffffff


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_f_init2 = _sig(_mpfr, "mpfr_init2", None, _PF, c_long)
_f_clear = _sig(_mpfr, "mpfr_clear", None, _PF)
_f_set = _sig(_mpfr, "mpfr_set", c_int, _PF, _PF, c_int)
_f_set_str = _sig(_mpfr, "mpfr_set_str", c_int, _PF, c_char_p, c_int, c_int)
_f_set_d = _sig(_mpfr, "mpfr_set_d", c_int, _PF, c_double, c_int)
_f_set_zero = _sig(_mpfr, "mpfr_set_zero", None, _PF, c_int)
_f_get_d = _sig(_mpfr, "mpfr_get_d", c_double, _PF, c_int)
_f_get_str = _sig(_mpfr, "mpfr_get_str", c_void_p, c_char_p, POINTER(c_long), c_int, c_size_t, _PF, c_int)
_f_free_str = _sig(_mpfr, "mpfr_free_str", None, c_void_p)
_f_cmp = _sig(_mpfr, "mpfr_cmp", c_int, _PF, _PF)
_f_zero_p = _sig(_mpfr, "mpfr_zero_p", c_int, _PF)
_f_signbit = _sig(_mpfr, "mpfr_signbit", c_int, _PF)
_f_number_p = _sig(_mpfr, "mpfr_number_p", c_int, _PF)
_f_nan_p = _sig(_mpfr, "mpfr_nan_p", c_int, _PF)
_f_mul_2si = _sig(_mpfr, "mpfr_mul_2si", c_int, _PF, _PF, c_long, c_int)
_f_urandom = _sig(_mpfr, "mpfr_urandom", c_int, _PF, c_void_p, c_int)
_f_const_pi = _sig(_mpfr, "mpfr_const_pi", c_int, _PF, c_int)
_f_fac_ui = _sig(_mpfr, "mpfr_fac_ui", c_int, _PF, c_ulong, c_int)
_f_pow_si = _sig(_mpfr, "mpfr_pow_si", c_int, _PF, _PF, c_long, c_int)
_f_pow = _sig(_mpfr, "mpfr_pow", c_int, _PF, _PF, _PF, c_int)
_f_bin = {name: _sig(_mpfr, "mpfr_" + name, c_int, _PF, _PF, _PF, c_int)
          for name in ("add", "sub", "mul", "div")}
_f_un = {name: _sig(_mpfr, "mpfr_" + name, c_int, _PF, _PF, c_int)
         for name in ("neg", "abs", "exp", "log", "log2", "log10", "sqrt", "sin", "cos", "gamma")}

_c_init3 = _sig(_mpc, "mpc_init3", None, _PC, c_long, c_long)
_c_clear = _sig(_mpc, "mpc_clear", None, _PC)
_c_set_fr_fr = _sig(_mpc, "mpc_set_fr_fr", c_int, _PC, _PF, _PF, c_int)
_c_abs = _sig(_mpc, "mpc_abs", c_int, _PF, _PC, c_int)
_c_bin = {name: _sig(_mpc, "mpc_" + name, c_int, _PC, _PC, _PC, c_int)
          for name in ("add", "sub", "mul", "div", "pow")}
_c_un = {name: _sig(_mpc, "mpc_" + name, c_int, _PC, _PC, c_int)
         for name in ("neg", "exp", "log", "sqrt", "sin", "cos")}

_z_init = _sig(_gmp, "__gmpz_init", None, _PZ)
_z_clear = _sig(_gmp, "__gmpz_clear", None, _PZ)
_z_set_str = _sig(_gmp, "__gmpz_set_str", c_int, _PZ, c_char_p, c_int)
_r_init = _sig(_gmp, "__gmp_randinit_default", None, c_void_p)
_r_seed = _sig(_gmp, "__gmp_randseed", None, c_void_p, _PZ)
_r_clear = _sig(_gmp, "__gmp_randclear", None, c_void_p)

_RNDN = 0


# ------------------------------------------------------------------ context

class context:
    """gmpy2.context(precision=...) usable as a context manager."""

    def __init__(self, precision=53, **kw):
        self.precision = int(precision)
        self.real_prec = self.imag_prec = self.precision

    def __enter__(self):
        _ctx_stack().append(self)
        return self

    def __exit__(self, *exc):
        _ctx_stack().pop()
        return False

    def __repr__(self):
        return f"context(precision={self.precision})"


_tls = threading.local()


def _ctx_stack():
    st = getattr(_tls, "stack", None)
    if st is None:
        st = _tls.stack = [context(53)]
    return st


def get_context():
    return _ctx_stack()[-1]


def local_context(ctx=None, **kw):
    base = ctx or get_context()
    return context(kw.get("precision", base.precision))


def _prec():
    return get_context().precision


# ------------------------------------------------------------------ mpz / mpq

class mpz(int):
    def __new__(cls, v=0, base=10):
        if isinstance(v, str):
            return int.__new__(cls, int(v, base))
        return int.__new__(cls, int(v))


def mpq(n, d=1):
    return Fraction(int(n), int(d))


def _int_to_mpz(v: int):
    z = _MPZ_T()
    _z_init(byref(z))
    _z_set_str(byref(z), format(v, "x").encode() if v >= 0 else ("-" + format(-v, "x")).encode(), 16)
    return z


# ------------------------------------------------------------------ mpfr

def _new_raw(prec: int) -> "mpfr":
    obj = object.__new__(mpfr)
    s = _MPFR_T()
    _f_init2(byref(s), max(int(prec), 1))
    obj._s = s
    return obj


def _exact_from_int(v: int) -> "mpfr":
    bits = max(64, abs(v).bit_length())
    r = _new_raw(bits)
    txt = format(v, "x") if v >= 0 else "-" + format(-v, "x")
    _f_set_str(byref(r._s), txt.encode(), 16, _RNDN)
    return r


def _exact_from_float(v: float) -> "mpfr":
    r = _new_raw(64)
    _f_set_d(byref(r._s), v, _RNDN)
    return r


def _to_exact_mpfr(x):
    """Exact mpfr for a real operand (int/float/mpz/bool/mpfr)."""
    if isinstance(x, mpfr):
        return x
    if isinstance(x, bool):
        return _exact_from_int(int(x))
    if isinstance(x, int):
        return _exact_from_int(int(x))
    if isinstance(x, float):
        return _exact_from_float(x)
    return None


def _round_fraction(fr: Fraction, prec: int) -> "mpfr":
    num = _exact_from_int(fr.numerator)
    den = _exact_from_int(fr.denominator)
    r = _new_raw(prec)
    _f_bin["div"](byref(r._s), byref(num._s), byref(den._s), _RNDN)
    return r


class mpfr:
    __slots__ = ("_s", "__weakref__")

    def __new__(cls, x=0, precision=0, base=10):
        prec = int(precision) if precision else _prec()
        r = _new_raw(prec)
        if isinstance(x, mpfr):
            _f_set(byref(r._s), byref(x._s), _RNDN)
        elif isinstance(x, str):
            t = x.strip()
            if t in ("-0", "-0.0"):
                _f_set_zero(byref(r._s), -1)
            elif _f_set_str(byref(r._s), t.encode(), base, _RNDN) != 0:
                raise ValueError(f"invalid digits {x!r}")
        elif isinstance(x, Fraction):
            return _round_fraction(x, prec)
        elif isinstance(x, (int, float)):
            e = _to_exact_mpfr(x)
            _f_set(byref(r._s), byref(e._s), _RNDN)
        elif isinstance(x, mpc):
            raise TypeError("mpfr() of mpc")
        else:
            raise TypeError(f"mpfr() of {type(x).__name__}")
        return r

    def __del__(self):
        try:
            _f_clear(byref(self._s))
        except Exception:
            pass

    # -- attributes
    @property
    def precision(self):
        return int(self._s.prec)

    @property
    def real(self):
        return self

    @property
    def imag(self):
        return mpfr(0, self.precision)

    def is_zero(self):
        return bool(_f_zero_p(byref(self._s)))

    # values are immutable (as gmpy2's): copies are the object itself; pickling carries
    # the exact limbs and the precision
    def __copy__(self):
        return self

    def __deepcopy__(self, memo):
        return self

    def __reduce__(self):
        if not _f_number_p(byref(self._s)):  # NaN / Inf
            text = "@NaN@" if _f_nan_p(byref(self._s)) else ("-@Inf@" if _f_signbit(byref(self._s)) else "@Inf@")
            return (_mpfr_from_str, (text, self.precision))
        return (from_limbs, limbs_of(self) + (self.precision,))

    def as_mantissa_exp(self):
        if self.is_zero():
            return mpz(0), mpz(1)
        p = self.precision
        n64 = (p + 63) // 64
        mag = 0
        for k in range(n64 - 1, -1, -1):
            mag = (mag << 64) | int(self._s.d[k])
        mag >>= 64 * n64 - p
        e = int(self._s.exp) - p
        m = -mag if _f_signbit(byref(self._s)) else mag
        return mpz(m), mpz(e)

    def _fraction(self):
        if self.is_zero():
            return Fraction(0)
        m, e = self.as_mantissa_exp()
        return Fraction(int(m)) * (Fraction(2) ** int(e))

    def digits(self, base=10, prec=0):
        ex = c_long(0)
        ptr = _f_get_str(None, byref(ex), base, prec, byref(self._s), _RNDN)
        s = ctypes.string_at(ptr).decode()
        _f_free_str(ptr)
        return s, int(ex.value), self.precision

    # -- conversions
    def __float__(self):
        return float(_f_get_d(byref(self._s), _RNDN))

    def __int__(self):
        return int(self._fraction())

    def __bool__(self):
        return not self.is_zero()

    def __hash__(self):
        return hash(self._fraction())

    def __repr__(self):
        return f"mpfr('{_fmt(self)}',{self.precision})"

    def __str__(self):
        return _fmt(self)

    # -- arithmetic
    def _bin(self, other, op, rev=False):
        if isinstance(other, (mpc, complex)):
            a, b = mpc(self), mpc(other)
            return a._bin(b, op) if not rev else b._bin(a, op)
        if isinstance(other, Fraction):
            o = _round_fraction(other, max(_prec(), 64) + 256)  # operands of rational ops
        else:
            o = _to_exact_mpfr(other)
        if o is None:
            return NotImplemented
        a, b = (o, self) if rev else (self, o)
        r = _new_raw(_prec())
        _f_bin[op](byref(r._s), byref(a._s), byref(b._s), _RNDN)
        return r

    def __add__(self, o): return self._bin(o, "add")
    def __radd__(self, o): return self._bin(o, "add", True)
    def __sub__(self, o): return self._bin(o, "sub")
    def __rsub__(self, o): return self._bin(o, "sub", True)
    def __mul__(self, o): return self._bin(o, "mul")
    def __rmul__(self, o): return self._bin(o, "mul", True)
    def __truediv__(self, o): return self._bin(o, "div")
    def __rtruediv__(self, o): return self._bin(o, "div", True)

    def __neg__(self):
        r = _new_raw(_prec())
        _f_un["neg"](byref(r._s), byref(self._s), _RNDN)
        return r

    def __pos__(self):
        return mpfr(self)

    def __abs__(self):
        r = _new_raw(_prec())
        _f_un["abs"](byref(r._s), byref(self._s), _RNDN)
        return r

    def __pow__(self, e):
        r = _new_raw(_prec())
        if isinstance(e, int):
            _f_pow_si(byref(r._s), byref(self._s), int(e), _RNDN)
        else:
            ee = _to_exact_mpfr(e)
            _f_pow(byref(r._s), byref(self._s), byref(ee._s), _RNDN)
        return r

    def __rpow__(self, b):
        return _to_exact_mpfr(b).__pow__(self)

    # -- comparison (exact)
    def _cmp(self, other):
        if isinstance(other, mpfr):
            return _f_cmp(byref(self._s), byref(other._s))
        if isinstance(other, (int, float)):
            if isinstance(other, float) and (math.isnan(other) or math.isinf(other)):
                return None
            o = _to_exact_mpfr(other)
            return _f_cmp(byref(self._s), byref(o._s))
        if isinstance(other, Fraction):
            a = self._fraction()
            return (a > other) - (a < other)
        return None

    def __eq__(self, o):
        if isinstance(o, (mpc, complex)):
            return mpc(self) == o
        c = self._cmp(o)
        return NotImplemented if c is None else c == 0

    def __ne__(self, o):
        r = self.__eq__(o)
        return r if r is NotImplemented else not r

    def __lt__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c < 0

    def __le__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c <= 0

    def __gt__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c > 0

    def __ge__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c >= 0


def _fmt(x: "mpfr") -> str:
    if x.is_zero():
        return "-0.0" if _f_signbit(byref(x._s)) else "0.0"
    d, e, _ = x.digits(10, 0)
    sign = ""
    if d.startswith("-"):
        sign, d = "-", d[1:]
    return f"{sign}0.{d}e{e}"


# ------------------------------------------------------------------ mpc

def _new_c(prec: int) -> "mpc":
    obj = object.__new__(mpc)
    s = _MPC_T()
    _c_init3(byref(s), prec, prec)
    obj._s = s
    return obj


def _exact_mpc(x):
    if isinstance(x, mpc):
        return x
    if isinstance(x, complex):
        re, im = _exact_from_float(x.real), _exact_from_float(x.imag)
    else:
        re = _to_exact_mpfr(x) if not isinstance(x, Fraction) else _round_fraction(x, _prec() + 256)
        if re is None:
            return None
        im = _exact_from_int(0)
    prec = max(re.precision, im.precision)
    r = _new_c(prec)
    _c_set_fr_fr(byref(r._s), byref(re._s), byref(im._s), 0)
    return r


class mpc:
    __slots__ = ("_s", "__weakref__")

    def __new__(cls, x=0, y=None, precision=0):
        prec = int(precision) if precision else _prec()
        if y is not None:
            re = x if isinstance(x, mpfr) else mpfr(x, 1 << 20) if not isinstance(x, (int, float)) else _to_exact_mpfr(x)
            im = y if isinstance(y, mpfr) else mpfr(y, 1 << 20) if not isinstance(y, (int, float)) else _to_exact_mpfr(y)
            r = _new_c(prec)
            _c_set_fr_fr(byref(r._s), byref(re._s), byref(im._s), 0)
            return r
        if isinstance(x, str):
            parts = x.replace("(", "").replace(")", "").split()
            return mpc(mpfr(parts[0]), mpfr(parts[1]) if len(parts) > 1 else 0, precision=prec)
        e = _exact_mpc(x)
        if e is None:
            raise TypeError(f"mpc() of {type(x).__name__}")
        r = _new_c(prec)
        _c_set_fr_fr(byref(r._s), byref(e._s.re), byref(e._s.im), 0)
        return r

    def __del__(self):
        try:
            _c_clear(byref(self._s))
        except Exception:
            pass

    def _part(self, which):
        f = getattr(self._s, which)
        r = _new_raw(int(f.prec))
        _f_set(byref(r._s), byref(f), _RNDN)
        return r

    @property
    def real(self):
        return self._part("re")

    @property
    def imag(self):
        return self._part("im")

    @property
    def precision(self):
        return (int(self._s.re.prec), int(self._s.im.prec))

    def __copy__(self):
        return self

    def __deepcopy__(self, memo):
        return self

    def __reduce__(self):
        return (mpc_from_parts, (self.real, self.imag))

    def _bin(self, other, op, rev=False):
        o = _exact_mpc(other)
        if o is None:
            return NotImplemented
        a, b = (o, self) if rev else (self, o)
        r = _new_c(_prec())
        _c_bin[op](byref(r._s), byref(a._s), byref(b._s), 0)
        return r

    def __add__(self, o): return self._bin(o, "add")
    def __radd__(self, o): return self._bin(o, "add", True)
    def __sub__(self, o): return self._bin(o, "sub")
    def __rsub__(self, o): return self._bin(o, "sub", True)
    def __mul__(self, o): return self._bin(o, "mul")
    def __rmul__(self, o): return self._bin(o, "mul", True)
    def __truediv__(self, o): return self._bin(o, "div")
    def __rtruediv__(self, o): return self._bin(o, "div", True)
    def __pow__(self, o): return self._bin(o, "pow")

    def __neg__(self):
        r = _new_c(_prec())
        _c_un["neg"](byref(r._s), byref(self._s), 0)
        return r

    def __abs__(self):
        r = _new_raw(_prec())
        _c_abs(byref(r._s), byref(self._s), _RNDN)
        return r

    def __eq__(self, o):
        o2 = _exact_mpc(o)
        if o2 is None:
            return NotImplemented
        return self.real == o2.real and self.imag == o2.imag

    def __ne__(self, o):
        r = self.__eq__(o)
        return r if r is NotImplemented else not r

    def __bool__(self):
        return bool(self.real) or bool(self.imag)

    def __hash__(self):
        return hash((hash(self.real), hash(self.imag)))

    def __complex__(self):
        return complex(float(self.real), float(self.imag))

    def __repr__(self):
        return f"mpc('{_fmt(self.real)} {_fmt(self.imag)}')"


# ------------------------------------------------------------------ functions

def _unary(name, x):
    if isinstance(x, (mpc, complex)):
        a = _exact_mpc(x)
        r = _new_c(_prec())
        _c_un[name](byref(r._s), byref(a._s), 0)
        return r
    a = _to_exact_mpfr(x) if not isinstance(x, Fraction) else _round_fraction(x, _prec())
    r = _new_raw(_prec())
    _f_un[name](byref(r._s), byref(a._s), _RNDN)
    return r


def exp(x): return _unary("exp", x)
def log(x): return _unary("log", x)
def sqrt(x): return _unary("sqrt", x)
def sin(x): return _unary("sin", x)
def cos(x): return _unary("cos", x)
def log2(x): return _unary("log2", x)
def log10(x): return _unary("log10", x)
def gamma(x): return _unary("gamma", x)


def const_pi(precision=0):
    r = _new_raw(int(precision) if precision else _prec())
    _f_const_pi(byref(r._s), _RNDN)
    return r


def factorial(k):
    r = _new_raw(_prec())
    _f_fac_ui(byref(r._s), int(k), _RNDN)
    return r


def is_finite(x):
    if isinstance(x, mpc):
        return is_finite(x.real) and is_finite(x.imag)
    if isinstance(x, mpfr):
        return bool(_f_number_p(byref(x._s)))
    return math.isfinite(x)


def is_signed(x):
    if isinstance(x, mpfr):
        return bool(_f_signbit(byref(x._s)))
    return math.copysign(1.0, float(x)) < 0


def is_zero(x):
    return x == 0


def mul_2exp(x, n):
    a = x if isinstance(x, mpfr) else mpfr(x)
    r = _new_raw(_prec())
    _f_mul_2si(byref(r._s), byref(a._s), int(n), _RNDN)
    return r


def div_2exp(x, n):
    return mul_2exp(x, -int(n))


class random_state:
    def __init__(self, seed=0):
        self._buf = ctypes.create_string_buffer(128)
        _r_init(self._buf)
        z = _int_to_mpz(int(seed))
        _r_seed(self._buf, byref(z))
        _z_clear(byref(z))

    def __del__(self):
        try:
            _r_clear(self._buf)
        except Exception:
            pass


def mpfr_random(state):
    r = _new_raw(_prec())
    _f_urandom(byref(r._s), state._buf, _RNDN)
    return r


# ------------------------------------------------------------------ SoA glue
# Fast conversion between these objects and the ds SoA limb format
# (include/detseries_b200.h): 32-bit little-endian limbs, left-aligned.

def limbs_of(x: "mpfr"):
    """(limb bytes (little-endian, 4L bytes), exp, cls) of a real scalar."""
    p = x.precision
    L = (p + 31) // 32
    if x.is_zero():
        return bytes(4 * L), 0, (3 if _f_signbit(byref(x._s)) else 2)
    n64 = (p + 63) // 64
    raw = ctypes.string_at(x._s.d, 8 * n64)
    if 2 * n64 != L:  # drop the low 32 padding bits
        raw = raw[4:]
    return raw, int(x._s.exp), (1 if _f_signbit(byref(x._s)) else 0)


def _mpfr_from_str(text: str, prec: int) -> "mpfr":
    return mpfr(text, prec)


def from_limbs(raw: bytes, exp: int, cls: int, prec: int) -> "mpfr":
    """Inverse of limbs_of: build an mpfr of precision `prec` (exact)."""
    r = _new_raw(prec)
    if cls >= 2:
        _f_set_zero(byref(r._s), -1 if cls == 3 else 1)
        return r
    L = (prec + 31) // 32
    n64 = (prec + 63) // 64
    if 2 * n64 != L:
        raw = bytes(4) + raw
    ctypes.memmove(r._s.d, raw, 8 * n64)
    r._s.exp = int(exp)
    r._s.sign = -1 if cls == 1 else 1
    return r


class _pooled_mpfr(mpfr):
    """mpfr over struct k of a ctypes array of initialised structs whose significands
    live in a shared limb pool (SoA.scalars, hostgen.RowQueue).  The object holds the
    array (which holds the pool's owner); the struct view is made on access, so
    creating one costs two slot stores and nothing is freed per scalar.  Behaves as
    mpfr everywhere (isinstance, arithmetic, formatting)."""
    __slots__ = ("_arr", "_k")

    @property
    def _s(self):
        return self._arr[self._k]

    def __del__(self):
        pass


def wrap_pooled(arr, owner, count: int) -> list:
    """Scalars over arr[0..count); `owner` (the limb pool / native batch) lives as long
    as any of them."""
    arr._owner = owner
    new = object.__new__
    out = []
    for k in range(count):
        o = new(_pooled_mpfr)
        o._arr = arr
        o._k = k
        out.append(o)
    return out


def mpc_from_parts(re: "mpfr", im: "mpfr") -> "mpc":
    """Exact complex from two reals of the same precision."""
    r = _new_c(re.precision)
    _c_set_fr_fr(byref(r._s), byref(re._s), byref(im._s), 0)
    return r

"""CPU oracle for the CKKS encrypted-dense-layer hot path (arXiv 2205.11935).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
(and `--impl reference`) leg may import this package.  The product package
`paper_2205_11935_b200` never imports it, and this package never imports the product.

Layout:
  ckks_oracle.c  -- scalar C: primes, psi, textbook NTT, automorphism, PRNG/samplers, keys,
                    encrypt/decrypt, key switch, rotate, relinearize, rescale (fp-free).
  encoding.py    -- fp64 canonical-embedding encode/decode and big-integer CRT lift (numpy FFT).
  circuits.py    -- BSGS dense layer (Eq. 1), activations (square, Eq. 2), replicate, forward,
                    and the float64 plaintext reference forward.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ckks_oracle.c")
_BUILD = os.path.join(_HERE, "_build")
_SO = os.path.join(_BUILD, "libckks_oracle.so")


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, no vectorisation flags)."""
    os.makedirs(_BUILD, exist_ok=True)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
i8p = ctypes.POINTER(ctypes.c_int8)
vp = ctypes.c_void_p
U64, I64, INT, DBL = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_double


def _declare(L):
    sig = {
        "or_ctx_new": (vp, [INT, INT, INT, ctypes.POINTER(ctypes.c_int), DBL]),
        "or_ctx_new_primes": (vp, [INT, INT, INT, u64p, DBL]),
        "or_ctx_free": (None, [vp]),
        "or_set_digits": (INT, [vp, ctypes.POINTER(ctypes.c_int), INT]),
        "or_n_digits": (INT, [vp]),
        "or_n_special": (INT, [vp]),
        "or_n": (INT, [vp]),
        "or_n_data": (INT, [vp]),
        "or_prime": (U64, [vp, INT]),
        "or_psi": (U64, [vp, INT]),
        "or_prng": (U64, [U64, U64, U64]),
        "or_stream": (U64, [U64, U64, U64, U64]),
        "or_sample_ternary": (None, [U64, U64, i8p, I64]),
        "or_sample_uniform": (None, [U64, U64, U64, u64p, I64]),
        "or_sample_gaussian": (None, [vp, U64, U64, i64p, I64]),
        "or_cdt": (U64, [vp, INT]),
        "or_cdt_bound": (INT, [vp]),
        "or_ntt": (None, [vp, INT, u64p]),
        "or_intt": (None, [vp, INT, u64p]),
        "or_automorphism_coef": (None, [vp, INT, u64p, U64, u64p]),
        "or_automorphism_ntt": (None, [vp, INT, u64p, U64, u64p]),
        "or_galois_elt": (U64, [vp, I64]),
        "or_keygen": (INT, [vp, U64]),
        "or_gen_switch_key": (INT, [vp, U64, I64]),
        "or_export_key": (INT, [vp, I64, u64p]),
        "or_export_secret": (INT, [vp, i8p]),
        "or_export_pk": (INT, [vp, u64p]),
        "or_plain_from_coeffs": (None, [vp, i64p, INT, u64p]),
        "or_encrypt": (INT, [vp, i64p, U64, U64, u64p]),
        "or_decrypt": (INT, [vp, u64p, INT, u64p]),
        "or_add": (None, [vp, u64p, u64p, INT, INT, u64p]),
        "or_mul_plain": (None, [vp, u64p, u64p, INT, u64p]),
        "or_add_plain": (None, [vp, u64p, u64p, INT, u64p]),
        "or_tensor": (None, [vp, u64p, u64p, INT, u64p]),
        "or_keyswitch": (INT, [vp, u64p, INT, I64, u64p]),
        "or_relinearize": (INT, [vp, u64p, INT, u64p]),
        "or_rotate": (INT, [vp, u64p, INT, I64, u64p]),
        "or_rotate_hoisted": (INT, [vp, u64p, INT, I64, u64p]),
        "or_rotate_hoisted_qp": (INT, [vp, u64p, INT, I64, u64p]),
        "or_rotate_qp": (INT, [vp, u64p, INT, I64, u64p]),
        "or_moddown": (None, [vp, u64p, INT, INT, u64p]),
        "or_lift_qp": (None, [vp, u64p, INT, INT, u64p]),
        "or_plain_qp": (None, [vp, i64p, INT, u64p]),
        "or_mul_plain_qp": (None, [vp, u64p, u64p, INT, u64p]),
        "or_add_qp": (None, [vp, u64p, u64p, INT, INT, u64p]),
        "or_rescale": (INT, [vp, u64p, INT, INT, u64p]),
        "or_drop_level": (None, [vp, u64p, INT, INT, INT, u64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _p(a, t=u64p):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    pass


def _check(st, what):
    if st != 0:
        raise OracleError(f"{what} failed with status {st}")


class Context:
    """Oracle CKKS context: prime chain, tables, and (after keygen) the seeded keys."""

    def __init__(self, log_n, data_bits, special_bits=(), sigma=3.2, primes=None, digits=None):
        """digits: sizes of the key-switching digits (consecutive data primes, R9b), default one per prime."""
        L = lib()
        self.log_n = int(log_n)
        self.n = 1 << self.log_n
        self.n_data = len(data_bits) if primes is None else len(primes) - len(special_bits)
        self.n_special = len(special_bits)
        if primes is None:
            bits = (ctypes.c_int * (self.n_data + self.n_special))(*data_bits, *special_bits)
            self._c = L.or_ctx_new(self.log_n, self.n_data, self.n_special, bits, sigma)
        else:
            arr = np.ascontiguousarray(np.array(primes, dtype=np.uint64))
            self._arr = arr
            self._c = L.or_ctx_new_primes(self.log_n, self.n_data, self.n_special, _p(arr), sigma)
        if not self._c:
            raise OracleError("or_ctx_new failed (bad parameters)")
        if digits is not None:
            arr = (ctypes.c_int * len(digits))(*[int(d) for d in digits])
            _check(L.or_set_digits(self._c, arr, len(digits)), "set_digits")
        self.n_digits = int(L.or_n_digits(self._c))
        self.digits = list(digits) if digits is not None else [1] * self.n_data
        self.primes = [int(L.or_prime(self._c, i)) for i in range(self.n_data + self.n_special)]
        self.psi = [int(L.or_psi(self._c, i)) for i in range(self.n_data + self.n_special)]
        self.keys = set()
        self.key_seed = None

    def __del__(self):
        if getattr(self, "_c", None):
            lib().or_ctx_free(self._c)
            self._c = None

    @property
    def special(self):
        return self.primes[self.n_data] if self.n_special else None

    @property
    def special_product(self):
        P = 1
        for q in self.primes[self.n_data:]:
            P *= q
        return P

    @property
    def top_level(self):
        return self.n_data - 1

    # ---------------------------------------------------------------- ring
    def ntt(self, a, pi):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().or_ntt(self._c, pi, _p(a))
        return a

    def intt(self, a, pi):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().or_intt(self._c, pi, _p(a))
        return a

    def automorphism_coef(self, a, pi, g):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = np.empty_like(a)
        lib().or_automorphism_coef(self._c, pi, _p(a), g, _p(out))
        return out

    def automorphism_ntt(self, a, pi, g):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = np.empty_like(a)
        lib().or_automorphism_ntt(self._c, pi, _p(a), g, _p(out))
        return out

    def galois_elt(self, step):
        return int(lib().or_galois_elt(self._c, step))

    # ---------------------------------------------------------------- samplers
    def sample_gaussian(self, seed, stream, count):
        out = np.empty(count, dtype=np.int64)
        lib().or_sample_gaussian(self._c, seed, stream, _p(out, i64p), count)
        return out

    def cdt(self):
        B = lib().or_cdt_bound(self._c)
        return [int(lib().or_cdt(self._c, k)) for k in range(2 * B)], B

    # ---------------------------------------------------------------- keys
    def keygen(self, seed, rot_steps=(), relin=True):
        _check(lib().or_keygen(self._c, seed), "keygen")
        self.key_seed = seed
        if relin:
            self.add_switch_key(0)
        for st in rot_steps:
            g = self.galois_elt(st)
            if g != 1:
                self.add_switch_key(g)

    def add_switch_key(self, key_id):
        _check(lib().or_gen_switch_key(self._c, self.key_seed, key_id), "gen_switch_key")
        self.keys.add(int(key_id))

    def export_key(self, key_id):
        L = self.n_data
        out = np.empty((self.n_digits, 2, L + self.n_special, self.n), dtype=np.uint64)
        _check(lib().or_export_key(self._c, key_id, _p(out)), "export_key")
        return out

    def export_secret(self):
        out = np.empty(self.n, dtype=np.int8)
        _check(lib().or_export_secret(self._c, _p(out, i8p)), "export_secret")
        return out

    def export_pk(self):
        out = np.empty((2, self.n_data, self.n), dtype=np.uint64)
        _check(lib().or_export_pk(self._c, _p(out)), "export_pk")
        return out

    # ---------------------------------------------------------------- scheme
    def plain(self, m_coeffs, level):
        m = np.ascontiguousarray(m_coeffs, dtype=np.int64)
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        lib().or_plain_from_coeffs(self._c, _p(m, i64p), level, _p(out))
        return out

    def encrypt(self, m_coeffs, enc_seed, index=0):
        m = np.ascontiguousarray(m_coeffs, dtype=np.int64)
        out = np.empty((2, self.n_data, self.n), dtype=np.uint64)
        _check(lib().or_encrypt(self._c, _p(m, i64p), enc_seed, index, _p(out)), "encrypt")
        return out

    def decrypt(self, ct):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        if ct.shape[0] != 2:
            raise OracleError("decrypt takes a size-2 ciphertext (S:L168)")
        level = ct.shape[1] - 1
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        _check(lib().or_decrypt(self._c, _p(ct), level, _p(out)), "decrypt")
        return out

    def add(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        assert a.shape == b.shape
        out = np.empty_like(a)
        lib().or_add(self._c, _p(a), _p(b), a.shape[1] - 1, a.shape[0], _p(out))
        return out

    def mul_plain(self, ct, pt):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        pt = np.ascontiguousarray(pt, dtype=np.uint64)
        assert pt.shape[0] == ct.shape[1]
        out = np.empty_like(ct)
        lib().or_mul_plain(self._c, _p(ct), _p(pt), ct.shape[1] - 1, _p(out))
        return out

    def add_plain(self, ct, pt):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        pt = np.ascontiguousarray(pt, dtype=np.uint64)
        assert pt.shape[0] == ct.shape[1]
        out = np.empty_like(ct)
        lib().or_add_plain(self._c, _p(ct), _p(pt), ct.shape[1] - 1, _p(out))
        return out

    def tensor(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.empty((3,) + a.shape[1:], dtype=np.uint64)
        lib().or_tensor(self._c, _p(a), _p(b), a.shape[1] - 1, _p(out))
        return out

    def keyswitch(self, d, key_id):
        d = np.ascontiguousarray(d, dtype=np.uint64)
        level = d.shape[0] - 1
        out = np.empty((2, level + 1, self.n), dtype=np.uint64)
        _check(lib().or_keyswitch(self._c, _p(d), level, key_id, _p(out)), "keyswitch")
        return out

    def relinearize(self, ct3):
        ct3 = np.ascontiguousarray(ct3, dtype=np.uint64)
        level = ct3.shape[1] - 1
        out = np.empty((2, level + 1, self.n), dtype=np.uint64)
        _check(lib().or_relinearize(self._c, _p(ct3), level, _p(out)), "relinearize")
        return out

    def rotate(self, ct, step):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty_like(ct)
        _check(lib().or_rotate(self._c, _p(ct), ct.shape[1] - 1, step, _p(out)), f"rotate({step})")
        return out

    def rotate_hoisted(self, ct, step):
        """Hoisted rotation (NEXT f-1): digits of the unrotated c1, automorphism on the signed digits."""
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty_like(ct)
        _check(lib().or_rotate_hoisted(self._c, _p(ct), ct.shape[1] - 1, step, _p(out)), f"rotate_hoisted({step})")
        return out

    # ---- QP basis (double hoisting, R11c): [ncomp][l+1+K][N], the last K limbs mod P_0..P_{K-1}
    def rotate_hoisted_qp(self, ct, step):
        """Baby step of R11c: hoisted rotation of a Q_l ciphertext left in the Q_l P basis."""
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        nl = ct.shape[1]
        out = np.empty((2, nl + self.n_special, self.n), dtype=np.uint64)
        _check(lib().or_rotate_hoisted_qp(self._c, _p(ct), nl - 1, step, _p(out)), f"rotate_hoisted_qp({step})")
        return out

    def rotate_qp(self, w, step):
        """Giant step of R11c: rotation of a Q_l P ciphertext, result in Q_l P."""
        w = np.ascontiguousarray(w, dtype=np.uint64)
        out = np.empty_like(w)
        _check(lib().or_rotate_qp(self._c, _p(w), w.shape[1] - 1 - self.n_special, step, _p(out)),
               f"rotate_qp({step})")
        return out

    def moddown(self, x):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        ncomp, ne = x.shape[0], x.shape[1]
        out = np.empty((ncomp, ne - self.n_special, self.n), dtype=np.uint64)
        lib().or_moddown(self._c, _p(x), ne - 1 - self.n_special, ncomp, _p(out))
        return out

    def lift_qp(self, ct):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        ncomp, nl = ct.shape[0], ct.shape[1]
        out = np.empty((ncomp, nl + self.n_special, self.n), dtype=np.uint64)
        lib().or_lift_qp(self._c, _p(ct), nl - 1, ncomp, _p(out))
        return out

    def plain_qp(self, coeffs, level):
        m = np.ascontiguousarray(coeffs, dtype=np.int64)
        out = np.empty((level + 1 + self.n_special, self.n), dtype=np.uint64)
        lib().or_plain_qp(self._c, _p(m, i64p), level, _p(out))
        return out

    def mul_plain_qp(self, ct, pt):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        pt = np.ascontiguousarray(pt, dtype=np.uint64)
        assert pt.shape[0] == ct.shape[1]
        out = np.empty_like(ct)
        lib().or_mul_plain_qp(self._c, _p(ct), _p(pt), ct.shape[1] - 1 - self.n_special, _p(out))
        return out

    def add_qp(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        assert a.shape == b.shape
        out = np.empty_like(a)
        lib().or_add_qp(self._c, _p(a), _p(b), a.shape[1] - 1 - self.n_special, a.shape[0], _p(out))
        return out

    def rescale(self, ct):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        ncomp, nl = ct.shape[0], ct.shape[1]
        out = np.empty((ncomp, nl - 1, self.n), dtype=np.uint64)
        _check(lib().or_rescale(self._c, _p(ct), nl - 1, ncomp, _p(out)), "rescale")
        return out

    def drop_level(self, ct, new_level):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        ncomp, nl = ct.shape[0], ct.shape[1]
        out = np.empty((ncomp, new_level + 1, self.n), dtype=np.uint64)
        lib().or_drop_level(self._c, _p(ct), nl - 1, new_level, ncomp, _p(out))
        return out


def prng(seed, stream, i):
    return int(lib().or_prng(seed, stream, i))


def stream(purpose, ident=0, digit=0, prime=0):
    return int(lib().or_stream(purpose, ident, digit, prime))


def sample_ternary(seed, strm, count):
    out = np.empty(count, dtype=np.int8)
    lib().or_sample_ternary(seed, strm, _p(out, i8p), count)
    return out


def sample_uniform(seed, strm, q, count):
    out = np.empty(count, dtype=np.uint64)
    lib().or_sample_uniform(seed, strm, q, _p(out), count)
    return out


from . import encoding  # noqa: E402,F401
from . import circuits  # noqa: E402,F401

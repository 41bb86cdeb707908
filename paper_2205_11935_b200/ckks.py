"""Thin ctypes binding of include/ckks.h (argument marshalling only).

Every function of the C-ABI is exposed under the same name (`ckks_ctx_create`, `ckks_ntt_fwd`, ...);
the classes below only allocate the caller-owned device buffers with torch and pass pointers.
No arithmetic of the method happens in Python, and there is no CPU fallback: if the shared
library is missing this module raises at import of `lib()`, and every compute call needs a GPU.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_lib = None

OK, E_PARAM, E_LEVEL, E_NOKEY, E_SCALE, E_DOMAIN, E_SHAPE, E_CUDA, E_SIZE = 0, -1, -2, -3, -4, -5, -6, -7, -8
ACT_NONE, ACT_SQUARE, ACT_CUBIC = 0, 1, 2


class CkksError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[ckks status {status}] {msg}")
        self.status = status


class ckks_params(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n_data", ctypes.c_uint32), ("n_special", ctypes.c_uint32),
                ("prime_bits", ctypes.POINTER(ctypes.c_uint32)), ("sigma", ctypes.c_double),
                ("key_seed", ctypes.c_uint64), ("rot_steps", ctypes.POINTER(ctypes.c_int32)),
                ("n_rot_steps", ctypes.c_uint32), ("want_relin", ctypes.c_int32), ("max_batch", ctypes.c_uint32),
                ("bsgs_baby_extra", ctypes.c_uint32), ("digit_sizes", ctypes.POINTER(ctypes.c_uint32)),
                ("n_digits", ctypes.c_uint32)]


class ckks_info(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n", ctypes.c_uint32), ("n_data", ctypes.c_uint32),
                ("n_special", ctypes.c_uint32), ("n_keys", ctypes.c_uint32),
                ("primes", ctypes.c_uint64 * 16), ("psi", ctypes.c_uint64 * 16), ("n_digits", ctypes.c_uint32),
                ("digit_sizes", ctypes.c_uint32 * 16)]


class ckks_ct(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("batch", ctypes.c_uint32), ("n_comp", ctypes.c_uint32),
                ("level", ctypes.c_uint32), ("scale", ctypes.c_double)]


class ckks_layer_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("rows", ctypes.c_uint32), ("cols", ctypes.c_uint32),
                ("t", ctypes.c_uint32), ("t2", ctypes.c_uint32), ("n_baby", ctypes.c_uint32),
                ("baby_steps", ctypes.POINTER(ctypes.c_int32)), ("giant", ctypes.c_int32),
                ("region", ctypes.c_uint32), ("items", ctypes.c_uint32), ("level", ctypes.c_uint32),
                ("pt_scale", ctypes.c_double), ("bias_scale", ctypes.c_double)]


class ckks_stage(ctypes.Structure):
    _fields_ = [("layer", ctypes.c_void_p), ("activation", ctypes.c_int32), ("replicate_t", ctypes.c_uint32)]


LAYER_DENSE, LAYER_CONV1D, LAYER_AVGPOOL = 0, 1, 2

_VP, _SZ = ctypes.c_void_p, ctypes.c_size_t
_PSZ = ctypes.POINTER(ctypes.c_size_t)
_PCT = ctypes.POINTER(ckks_ct)
_I, _U32, _U64, _I64, _D = ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double

SIGNATURES = {
    "ckks_last_error": (ctypes.c_char_p, []),
    "ckks_ctx_sizes": (_I, [ctypes.POINTER(ckks_params), _PSZ, _PSZ, _PSZ]),
    "ckks_ctx_create": (_I, [ctypes.POINTER(ckks_params), _VP, _VP, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_ctx_destroy": (None, [_VP]),
    "ckks_ctx_info": (_I, [_VP, ctypes.POINTER(ckks_info)]),
    "ckks_launch_count": (_U64, [_VP]),
    "ckks_set_option": (_I, [ctypes.c_char_p, _I64]),
    "ckks_get_option": (_I, [ctypes.c_char_p, ctypes.POINTER(_I64)]),
    "ckks_ntt_fwd": (_I, [_VP, _VP, _U32, _U32, _VP]),
    "ckks_ntt_inv": (_I, [_VP, _VP, _U32, _U32, _VP]),
    "ckks_rotate": (_I, [_VP, _PCT, _I, _PCT, _VP]),
    "ckks_mul": (_I, [_VP, _PCT, _PCT, _PCT, _VP]),
    "ckks_rotate_hoisted": (_I, [_VP, _PCT, ctypes.POINTER(_I), _U32, _PCT, _VP]),
    "ckks_dense_create_packed": (_I, [_VP, _VP, _U32, _U32, _VP, _U32, _U32, _U32, _D, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_conv1d_create": (_I, [_VP, _VP, _U32, _D, _U32, _U32, _U32, _U32, _D, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_avgpool_create": (_I, [_VP, _U32, _U32, _U32, _U32, _U32, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_layer_general_sizes": (_I, [_VP, _U32, _U32, _PSZ]),
    "ckks_layer_import_general": (_I, [_VP, ctypes.POINTER(ckks_layer_desc), _VP, _VP, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_model_stages_sizes": (_I, [_VP, ctypes.POINTER(ckks_stage), _U32, _PSZ]),
    "ckks_model_create_stages": (_I, [_VP, ctypes.POINTER(ckks_stage), _U32, _VP, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_model_set_hoisting": (_I, [_VP, _I]),
    "ckks_layer_set_hoisting": (_I, [_VP, _I]),
    "ckks_relinearize": (_I, [_VP, _PCT, _PCT, _VP]),
    "ckks_rescale": (_I, [_VP, _PCT, _PCT, _VP]),
    "ckks_add": (_I, [_VP, _PCT, _PCT, _PCT, _VP]),
    "ckks_layer_sizes": (_I, [_VP, _U32, _U32, _U32, _PSZ]),
    "ckks_layer_create": (_I, [_VP, _VP, _U32, _U32, _VP, _U32, _D, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_layer_import": (_I, [_VP, _VP, _VP, _U32, _U32, _U32, _D, _D, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_layer_destroy": (None, [_VP]),
    "ckks_layer_work_sizes": (_I, [_VP, _VP, _U32, _PSZ]),
    "ckks_matvec_diag": (_I, [_VP, _VP, _PCT, _PCT, _VP, _VP]),
    "ckks_model_sizes": (_I, [_VP, _U32, _I, _PSZ]),
    "ckks_model_create": (_I, [_VP, ctypes.POINTER(_VP), _U32, _I, _VP, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_model_destroy": (None, [_VP]),
    "ckks_model_work_sizes": (_I, [_VP, _VP, _U32, _PSZ]),
    "ckks_model_steps": (_I, [_U32, ctypes.POINTER(_U32), ctypes.POINTER(_U32), _U32, ctypes.POINTER(_I),
                              ctypes.POINTER(_U32)]),
    "ckks_model_levels": (_I, [_VP, ctypes.POINTER(_U32), ctypes.POINTER(_U32)]),
    "ckks_forward_graph_create": (_I, [_VP, _VP, _PCT, _PCT, _VP, _VP, ctypes.POINTER(_VP)]),
    "ckks_graph_launch": (_I, [_VP, _VP]),
    "ckks_graph_destroy": (None, [_VP]),
    "ckks_encrypted_forward": (_I, [_VP, _VP, _PCT, _PCT, _VP, _VP]),
    "ckks_encrypted_forward_host": (_I, [_VP, _VP, _VP, _U32, _U32, _D, _VP, ctypes.POINTER(_U32),
                                         ctypes.POINTER(_D), _VP, _VP]),
    "ckks_encode": (_I, [_VP, _VP, _U32, _D, _VP]),
    "ckks_encrypt": (_I, [_VP, _VP, _U32, _U64, _U64, _D, _PCT, _VP]),
    "ckks_encode_device": (_I, [_VP, _VP, _U32, _SZ, _U32, _D, _VP, _VP]),
    "ckks_encrypt_device": (_I, [_VP, _VP, _U32, _U64, _U64, _D, _PCT, _VP]),
    "ckks_decode_device": (_I, [_VP, _VP, _U32, _U32, _D, _VP, _U32, _VP]),
    "ckks_decrypt": (_I, [_VP, _PCT, _VP, _VP]),
    "ckks_decode": (_I, [_VP, _VP, _U32, _D, _VP, _U32]),
    "ckks_export_key": (_I, [_VP, _I64, _VP, _VP]),
    "ckks_galois_elt": (_U64, [_VP, _I]),
    "ckks_probe_enable": (_I, [_VP, _I]),
    "ckks_probe_read": (_I, [_VP, ctypes.POINTER(_D), ctypes.POINTER(_U64), ctypes.POINTER(_D)]),
    "ckks_probe_read_all": (_I, [_VP, ctypes.c_char_p, _SZ]),
    "ckks_bsgs_plan": (_I, [_U32, _U32, ctypes.POINTER(_U32), ctypes.POINTER(_U32), ctypes.POINTER(_U32)]),
    "ckks_bsgs_plan_x": (_I, [_U32, _U32, _U32, ctypes.POINTER(_U32), ctypes.POINTER(_U32), ctypes.POINTER(_U32)]),
    "ckks_model_plan": (_I, [_VP, _U32, ctypes.POINTER(_U32), ctypes.POINTER(_U32), _I, _U32, _D,
                             ctypes.POINTER(_U32), ctypes.POINTER(_D), ctypes.POINTER(_I), ctypes.POINTER(_U32)]),
}
PROBE_OFF, PROBE_MODUP, PROBE_KEYSWITCH, PROBE_NTT, PROBE_ALL = 0, 1, 2, 3, 4


def lib_path() -> str:
    return _build.LIB


def lib():
    """Load the in-tree shared library (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_build.LIB):
            raise ImportError(f"{_build.LIB} missing: run `python -m paper_2205_11935_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(_build.LIB)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status, what=""):
    if status != OK:
        msg = lib().ckks_last_error().decode(errors="replace")
        raise CkksError(status, f"{what}: {msg}")


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def u64_view(t):
    """torch int64 storage -> numpy uint64 array (copies to host)."""
    return t.detach().cpu().numpy().view(np.uint64)


class Ciphertext:
    """Device ciphertext batch: torch int64 tensor [batch][n_comp][level+1][N] holding u64 residues."""

    def __init__(self, data, level, scale, n_comp=2):
        self.data = data
        self.level = int(level)
        self.scale = float(scale)
        self.n_comp = int(n_comp)

    @property
    def batch(self):
        return int(self.data.shape[0])

    def c(self):
        return ckks_ct(ctypes.c_void_p(self.data.data_ptr()), self.batch, self.n_comp, self.level, self.scale)

    def numpy(self):
        return u64_view(self.data)


class Context:
    """Owns (as torch tensors) the table/key/workspace buffers that the C context borrows."""

    def __init__(self, log_n, data_bits, special_bits=(), key_seed=1, rot_steps=(), want_relin=True,
                 max_batch=1, sigma=3.2, device="cuda", stream=None, bsgs_baby_extra=0, digits=None):
        """digits: key-switching digit sizes (1 or 2 consecutive data primes each, R9b); None = one per prime."""
        import torch
        self.torch = torch
        self.device = torch.device(device)
        bits = list(data_bits) + list(special_bits)
        self._bits = (ctypes.c_uint32 * len(bits))(*bits)
        steps = [int(s) for s in rot_steps]
        self._steps = (ctypes.c_int32 * max(1, len(steps)))(*steps) if steps else (ctypes.c_int32 * 1)()
        self._digits = (ctypes.c_uint32 * len(digits))(*[int(d) for d in digits]) if digits else None
        self.params = ckks_params(int(log_n), len(data_bits), len(special_bits), self._bits, float(sigma),
                                  int(key_seed), self._steps, len(steps), 1 if want_relin else 0, int(max_batch),
                                  int(bsgs_baby_extra), self._digits, len(digits) if digits else 0)
        self.bsgs_baby_extra = int(bsgs_baby_extra)
        tb, kb, wb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().ckks_ctx_sizes(ctypes.byref(self.params), ctypes.byref(tb), ctypes.byref(kb),
                                    ctypes.byref(wb)), "ckks_ctx_sizes")
        self.tables = torch.empty(tb.value, dtype=torch.uint8, device=self.device)
        self.keys = torch.empty(kb.value, dtype=torch.uint8, device=self.device)
        self.work = torch.empty(wb.value, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _check(lib().ckks_ctx_create(ctypes.byref(self.params), _ptr(self.tables), _ptr(self.keys), _ptr(self.work),
                                     _stream(stream), ctypes.byref(h)), "ckks_ctx_create")
        self.h = h
        info = ckks_info()
        _check(lib().ckks_ctx_info(self.h, ctypes.byref(info)), "ckks_ctx_info")
        self.log_n, self.n = info.log_n, info.n
        self.n_data, self.n_special = info.n_data, info.n_special
        self.primes = [int(info.primes[i]) for i in range(self.n_data + self.n_special)]
        self.psi = [int(info.psi[i]) for i in range(self.n_data + self.n_special)]
        self.n_keys = info.n_keys
        self.max_batch = int(max_batch)
        self.n_digits = info.n_digits
        self.digits = [int(info.digit_sizes[j]) for j in range(self.n_digits)]

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().ckks_ctx_destroy(self.h)
            except Exception:
                pass
            self.h = None

    @property
    def top_level(self):
        return self.n_data - 1

    def launches(self):
        return int(lib().ckks_launch_count(self.h))

    def probe(self, kind):
        _check(lib().ckks_probe_enable(self.h, int(kind)), "ckks_probe_enable")

    def probe_read(self):
        ms, n, b = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_double()
        _check(lib().ckks_probe_read(self.h, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b)), "ckks_probe_read")
        return ms.value, n.value, b.value

    def probe_read_all(self):
        import json
        buf = ctypes.create_string_buffer(1 << 16)
        _check(lib().ckks_probe_read_all(self.h, buf, len(buf)), "ckks_probe_read_all")
        return json.loads(buf.value.decode())

    def model_plan(self, shapes, activation, in_level, in_scale):
        """-> ([layer input level], [layer input scale], [rotation steps]) from the library's planner."""
        k = len(shapes)
        rows = (_U32 * k)(*[r for r, _ in shapes])
        cols = (_U32 * k)(*[c for _, c in shapes])
        lv, sc, ns = (_U32 * k)(), (_D * k)(), _U32(0)
        _check(lib().ckks_model_plan(self.h, k, rows, cols, int(activation), int(in_level), float(in_scale), lv, sc,
                                     None, ctypes.byref(ns)), "ckks_model_plan")
        st = (_I * max(1, ns.value))()
        _check(lib().ckks_model_plan(self.h, k, rows, cols, int(activation), int(in_level), float(in_scale), lv, sc,
                                     st, ctypes.byref(ns)), "ckks_model_plan")
        return list(lv), list(sc), list(st[: ns.value])

    def galois_elt(self, step):
        return int(lib().ckks_galois_elt(self.h, int(step)))

    def empty_ct(self, batch, level, n_comp=2, scale=1.0):
        t = self.torch.empty((batch, n_comp, level + 1, self.n), dtype=self.torch.int64, device=self.device)
        return Ciphertext(t, level, scale, n_comp)

    def from_numpy(self, arr, level=None, scale=1.0):
        """Host u64 residues [batch][n_comp][l+1][N] -> device Ciphertext."""
        arr = np.ascontiguousarray(arr, dtype=np.uint64)
        if arr.ndim == 3:
            arr = arr[None]
        t = self.torch.from_numpy(arr.view(np.int64)).to(self.device)
        return Ciphertext(t, arr.shape[2] - 1 if level is None else level, scale, arr.shape[1])

    # ---------------------------------------------------------------- ring
    def ntt_fwd(self, t, stream=None):
        b, l = int(t.shape[0]), int(t.shape[1])
        _check(lib().ckks_ntt_fwd(self.h, _ptr(t), b, l, _stream(stream)), "ckks_ntt_fwd")

    def ntt_inv(self, t, stream=None):
        b, l = int(t.shape[0]), int(t.shape[1])
        _check(lib().ckks_ntt_inv(self.h, _ptr(t), b, l, _stream(stream)), "ckks_ntt_inv")

    # ---------------------------------------------------------------- evaluator
    def _op(self, name, *cts, out=None, stream=None, extra=()):
        ins = [ct.c() for ct in cts]
        o = out.c()
        args = [self.h] + [ctypes.byref(x) for x in ins[:1]] + list(extra) + \
            [ctypes.byref(x) for x in ins[1:]] + [ctypes.byref(o), _stream(stream)]
        _check(getattr(lib(), name)(*args), name)
        out.level, out.scale, out.n_comp = o.level, o.scale, o.n_comp
        return out

    def rotate(self, ct, step, out=None, stream=None):
        out = out or self.empty_ct(ct.batch, ct.level)
        return self._op("ckks_rotate", ct, out=out, stream=stream, extra=(int(step),))

    def rotate_hoisted(self, ct, steps, outs=None, stream=None):
        steps = [int(s) for s in steps]
        outs = outs or [self.empty_ct(ct.batch, ct.level) for _ in steps]
        arr = (ckks_ct * len(steps))(*[o.c() for o in outs])
        st = (_I * len(steps))(*steps)
        i = ct.c()
        _check(lib().ckks_rotate_hoisted(self.h, ctypes.byref(i), st, len(steps), arr, _stream(stream)),
               "ckks_rotate_hoisted")
        for o, a in zip(outs, arr):
            o.level, o.scale = a.level, a.scale
        return outs

    def mul(self, a, b, out=None, stream=None):
        out = out or self.empty_ct(a.batch, a.level, 3)
        return self._op("ckks_mul", a, b, out=out, stream=stream)

    def relinearize(self, ct3, out=None, stream=None):
        out = out or self.empty_ct(ct3.batch, ct3.level)
        return self._op("ckks_relinearize", ct3, out=out, stream=stream)

    def rescale(self, ct, out=None, stream=None):
        out = out or self.empty_ct(ct.batch, ct.level - 1 if ct.level > 0 else 0, ct.n_comp)
        return self._op("ckks_rescale", ct, out=out, stream=stream)

    def add(self, a, b, out=None, stream=None):
        out = out or self.empty_ct(a.batch, a.level, a.n_comp)
        return self._op("ckks_add", a, b, out=out, stream=stream)

    # ---------------------------------------------------------------- client helpers
    def encode(self, values, scale):
        v = np.ascontiguousarray(values, dtype=np.float64)
        out = np.empty(self.n, dtype=np.int64)
        _check(lib().ckks_encode(self.h, v.ctypes.data_as(ctypes.c_void_p), v.size, float(scale),
                                 out.ctypes.data_as(ctypes.c_void_p)), "ckks_encode")
        return out

    def encrypt(self, coeffs, enc_seed, first_index=0, scale=1.0, stream=None):
        m = np.ascontiguousarray(coeffs, dtype=np.int64)
        if m.ndim == 1:
            m = m[None]
        out = self.empty_ct(m.shape[0], self.top_level, scale=scale)
        o = out.c()
        _check(lib().ckks_encrypt(self.h, m.ctypes.data_as(ctypes.c_void_p), m.shape[0], int(enc_seed),
                                  int(first_index), float(scale), ctypes.byref(o), _stream(stream)), "ckks_encrypt")
        return out

    def encode_device(self, values, scale, out=None, stream=None):
        """values: device float64 tensor [batch][count] -> device int64 coefficients [batch][N] (f-4)."""
        v = values if values.dim() == 2 else values[None]
        B, count = int(v.shape[0]), int(v.shape[1])
        out = out if out is not None else self.torch.empty((B, self.n), dtype=self.torch.int64, device=self.device)
        _check(lib().ckks_encode_device(self.h, _ptr(v), count, int(v.stride(0)), B, float(scale), _ptr(out),
                                        _stream(stream)), "ckks_encode_device")
        return out

    def encrypt_device(self, coeffs, enc_seed, first_index=0, scale=1.0, out=None, stream=None):
        """device int64 coefficients [batch][N] -> top-level ciphertexts (device encryption, no host copies)."""
        B = int(coeffs.shape[0])
        out = out or self.empty_ct(B, self.top_level, scale=scale)
        o = out.c()
        _check(lib().ckks_encrypt_device(self.h, _ptr(coeffs), B, int(enc_seed), int(first_index), float(scale),
                                         ctypes.byref(o), _stream(stream)), "ckks_encrypt_device")
        out.level, out.scale = o.level, o.scale
        return out

    def decode_device(self, residues, level, scale, count, out=None, stream=None):
        """device decrypted residues [batch][level+1][N] -> device float64 slot values [batch][count]."""
        B = int(residues.shape[0])
        out = out if out is not None else self.torch.empty((B, count), dtype=self.torch.float64, device=self.device)
        _check(lib().ckks_decode_device(self.h, _ptr(residues), int(level), B, float(scale), _ptr(out), int(count),
                                        _stream(stream)), "ckks_decode_device")
        return out

    def decrypt(self, ct, stream=None):
        out = self.torch.empty((ct.batch, ct.level + 1, self.n), dtype=self.torch.int64, device=self.device)
        c = ct.c()
        _check(lib().ckks_decrypt(self.h, ctypes.byref(c), _ptr(out), _stream(stream)), "ckks_decrypt")
        return out

    def decode(self, residues, level, scale, count=None):
        r = np.ascontiguousarray(residues, dtype=np.uint64)
        count = self.n // 2 if count is None else count
        out = np.empty(count, dtype=np.float64)
        _check(lib().ckks_decode(self.h, r.ctypes.data_as(ctypes.c_void_p), int(level), float(scale),
                                 out.ctypes.data_as(ctypes.c_void_p), count), "ckks_decode")
        return out

    def export_key(self, key_id, stream=None):
        L = self.n_data
        if key_id == -1:
            shape = (L + self.n_special, self.n)
        elif key_id == -2:
            shape = (2, L, self.n)
        else:
            shape = (self.n_digits, 2, L + self.n_special, self.n)
        out = np.empty(shape, dtype=np.uint64)
        _check(lib().ckks_export_key(self.h, int(key_id), out.ctypes.data_as(ctypes.c_void_p), _stream(stream)),
               "ckks_export_key")
        return out


class Layer:
    """Encoded dense layer (device plaintexts owned here as a torch buffer)."""

    def __init__(self, ctx: Context, rows, cols, level, W=None, bias=None, in_scale=None, diag_coeffs=None,
                 bias_coeffs=None, pt_scale=None, bias_scale=None, stream=None):
        torch = ctx.torch
        self.ctx = ctx
        nb = ctypes.c_size_t()
        _check(lib().ckks_layer_sizes(ctx.h, rows, cols, level, ctypes.byref(nb)), "ckks_layer_sizes")
        self.buf = torch.empty(nb.value, dtype=torch.uint8, device=ctx.device)
        h = ctypes.c_void_p()
        if diag_coeffs is not None:
            d = np.ascontiguousarray(diag_coeffs, dtype=np.int64)
            b = None if bias_coeffs is None else np.ascontiguousarray(bias_coeffs, dtype=np.int64)
            self._keep = (d, b)
            _check(lib().ckks_layer_import(ctx.h, d.ctypes.data_as(ctypes.c_void_p),
                                           None if b is None else b.ctypes.data_as(ctypes.c_void_p), rows, cols,
                                           level, float(pt_scale), float(bias_scale), _ptr(self.buf),
                                           _stream(stream), ctypes.byref(h)), "ckks_layer_import")
        else:
            Wn = np.ascontiguousarray(W, dtype=np.float64)
            bn = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
            self._keep = (Wn, bn)
            _check(lib().ckks_layer_create(ctx.h, Wn.ctypes.data_as(ctypes.c_void_p), rows, cols,
                                           None if bn is None else bn.ctypes.data_as(ctypes.c_void_p), level,
                                           float(in_scale), _ptr(self.buf), _stream(stream), ctypes.byref(h)),
                   "ckks_layer_create")
        self.h = h
        self.level = level

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().ckks_layer_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def work_bytes(self, batch):
        nb = ctypes.c_size_t()
        _check(lib().ckks_layer_work_sizes(self.ctx.h, self.h, batch, ctypes.byref(nb)), "ckks_layer_work_sizes")
        return nb.value

    def set_hoisting(self, mode=1):
        """Rotation schedule of matvec: 0 none, 1 hoisted baby steps (R11b), 2 double hoisting (R11c)."""
        _check(lib().ckks_layer_set_hoisting(self.h, int(mode)), "ckks_layer_set_hoisting")
        return self

    def matvec(self, ct, out=None, work=None, stream=None):
        ctx = self.ctx
        out = out or ctx.empty_ct(ct.batch, ct.level - 1)
        if work is None:
            work = ctx.torch.empty(self.work_bytes(ct.batch), dtype=ctx.torch.uint8, device=ctx.device)
        i, o = ct.c(), out.c()
        _check(lib().ckks_matvec_diag(ctx.h, self.h, ctypes.byref(i), ctypes.byref(o), _ptr(work),
                                      _stream(stream)), "ckks_matvec_diag")
        out.level, out.scale = o.level, o.scale
        return out


class GeneralLayer(Layer):
    """Any f-2 layer (dense with item regions, conv1d, avgpool); built through the library encoder
    (`dense`, `conv1d`, `avgpool`) or imported from encoded coefficients (`imported`)."""

    def __init__(self, ctx, n_plaintexts, level, t, rows, build):
        torch = ctx.torch
        self.ctx = ctx
        nb = ctypes.c_size_t()
        _check(lib().ckks_layer_general_sizes(ctx.h, n_plaintexts, level, ctypes.byref(nb)), "ckks_layer_general_sizes")
        self.buf = torch.empty(nb.value, dtype=torch.uint8, device=ctx.device)
        h = ctypes.c_void_p()
        build(self, h)
        self.h = h
        self.level = level
        self.t = t
        self.rows = rows

    @classmethod
    def dense(cls, ctx, W, bias, region, items, level, in_scale, stream=None):
        Wn = np.ascontiguousarray(W, dtype=np.float64)
        rows, cols = Wn.shape
        t = bsgs_plan(rows, cols, ctx.bsgs_baby_extra)[0]
        bn = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)

        def build(self, h):
            self._keep = (Wn, bn)
            _check(lib().ckks_dense_create_packed(ctx.h, Wn.ctypes.data_as(ctypes.c_void_p), rows, cols,
                                                  None if bn is None else bn.ctypes.data_as(ctypes.c_void_p), region,
                                                  items, level, float(in_scale), _ptr(self.buf), _stream(stream),
                                                  ctypes.byref(h)), "ckks_dense_create_packed")
        return cls(ctx, t, level, t, rows, build)

    @classmethod
    def conv1d(cls, ctx, w, bias, t, region, items, level, in_scale, stream=None):
        wn = np.ascontiguousarray(w, dtype=np.float64)

        def build(self, h):
            self._keep = wn
            _check(lib().ckks_conv1d_create(ctx.h, wn.ctypes.data_as(ctypes.c_void_p), wn.size, float(bias), t, region,
                                            items, level, float(in_scale), _ptr(self.buf), _stream(stream),
                                            ctypes.byref(h)), "ckks_conv1d_create")
        return cls(ctx, wn.size, level, t, t, build)

    @classmethod
    def avgpool(cls, ctx, f, t, region, items, level, stream=None):
        def build(self, h):
            _check(lib().ckks_avgpool_create(ctx.h, f, t, region, items, level, _ptr(self.buf), _stream(stream),
                                             ctypes.byref(h)), "ckks_avgpool_create")
        return cls(ctx, f, level, t, t, build)

    @classmethod
    def imported(cls, ctx, kind, rows, cols, t, t2, baby_steps, giant, region, items, level, pt_scale, bias_scale,
                 pt_coeffs, bias_coeffs=None, stream=None):
        steps = (ctypes.c_int32 * len(baby_steps))(*[int(s) for s in baby_steps])
        pts = np.ascontiguousarray(pt_coeffs, dtype=np.int64)
        bc = None if bias_coeffs is None else np.ascontiguousarray(bias_coeffs, dtype=np.int64)
        d = ckks_layer_desc(kind, rows, cols, t, t2, len(baby_steps), steps, giant, region, items, level,
                            float(pt_scale), float(bias_scale))

        def build(self, h):
            self._keep = (steps, pts, bc, d)
            _check(lib().ckks_layer_import_general(ctx.h, ctypes.byref(d), pts.ctypes.data_as(ctypes.c_void_p),
                                                   None if bc is None else bc.ctypes.data_as(ctypes.c_void_p),
                                                   _ptr(self.buf), _stream(stream), ctypes.byref(h)),
                   "ckks_layer_import_general")
        return cls(ctx, pts.shape[0], level, t, rows, build)


class Model:
    def __init__(self, ctx: Context, layers, activation=ACT_SQUARE, act_coeffs=None, stream=None):
        self.ctx = ctx
        self.layers = list(layers)
        arr = (ctypes.c_void_p * len(layers))(*[l.h.value for l in layers])
        nb = ctypes.c_size_t()
        _check(lib().ckks_model_sizes(ctx.h, len(layers), int(activation), ctypes.byref(nb)), "ckks_model_sizes")
        self.buf = ctx.torch.empty(max(1, nb.value), dtype=ctx.torch.uint8, device=ctx.device)
        ac = None if act_coeffs is None else np.ascontiguousarray(act_coeffs, dtype=np.int64)
        self._keep = ac
        h = ctypes.c_void_p()
        _check(lib().ckks_model_create(ctx.h, arr, len(layers), int(activation),
                                       None if ac is None else ac.ctypes.data_as(ctypes.c_void_p), _ptr(self.buf),
                                       _stream(stream), ctypes.byref(h)), "ckks_model_create")
        self.h = h
        self._levels()

    def _levels(self):
        il, ol = _U32(), _U32()
        _check(lib().ckks_model_levels(self.h, ctypes.byref(il), ctypes.byref(ol)), "ckks_model_levels")
        self.in_level, self.final_level = il.value, ol.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().ckks_model_destroy(self.h)
            except Exception:
                pass
            self.h = None

    @classmethod
    def from_stages(cls, ctx, stages, act_coeffs=None, stream=None):
        """stages: [(layer, activation, replicate_t)]."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.layers = [s[0] for s in stages]
        arr = (ckks_stage * len(stages))(*[ckks_stage(l.h.value, int(a), int(r)) for l, a, r in stages])
        nb = ctypes.c_size_t()
        _check(lib().ckks_model_stages_sizes(ctx.h, arr, len(stages), ctypes.byref(nb)), "ckks_model_stages_sizes")
        self.buf = ctx.torch.empty(max(1, nb.value), dtype=ctx.torch.uint8, device=ctx.device)
        ac = None if act_coeffs is None else np.ascontiguousarray(act_coeffs, dtype=np.int64)
        self._keep = (ac, arr)
        h = ctypes.c_void_p()
        _check(lib().ckks_model_create_stages(ctx.h, arr, len(stages),
                                              None if ac is None else ac.ctypes.data_as(ctypes.c_void_p),
                                              _ptr(self.buf), _stream(stream), ctypes.byref(h)),
               "ckks_model_create_stages")
        self.h = h
        self._levels()
        return self

    def set_hoisting(self, mode=1):
        """0 none, 1 (or True) hoisted baby steps (R11b), 2 double hoisting (R11c)."""
        mode = int(mode)
        _check(lib().ckks_model_set_hoisting(self.h, mode), "ckks_model_set_hoisting")
        self.hoisted = mode

    def work_bytes(self, batch):
        nb = ctypes.c_size_t()
        _check(lib().ckks_model_work_sizes(self.ctx.h, self.h, batch, ctypes.byref(nb)), "ckks_model_work_sizes")
        return nb.value

    def forward(self, ct, out=None, work=None, stream=None):
        ctx = self.ctx
        if out is None:
            out = ctx.empty_ct(ct.batch, self.final_level)
        if work is None:
            work = ctx.torch.empty(self.work_bytes(ct.batch), dtype=ctx.torch.uint8, device=ctx.device)
        i, o = ct.c(), out.c()
        _check(lib().ckks_encrypted_forward(ctx.h, self.h, ctypes.byref(i), ctypes.byref(o), _ptr(work),
                                            _stream(stream)), "ckks_encrypted_forward")
        out.level, out.scale = o.level, o.scale
        return out

    def graph(self, ct, out=None, work=None, stream=None):
        """CUDA graph of the forward ct -> out (buffers bound at capture); replay with .launch()."""
        return ForwardGraph(self, ct, out, work, stream)

    def forward_host(self, h_in, in_level, in_scale, h_out, work, stream=None):
        """h_in / h_out: pinned torch int64 CPU tensors.  Returns (out_level, out_scale)."""
        ol, osc = ctypes.c_uint32(), ctypes.c_double()
        _check(lib().ckks_encrypted_forward_host(self.ctx.h, self.h, _ptr(h_in), int(h_in.shape[0]), int(in_level),
                                                 float(in_scale), _ptr(h_out), ctypes.byref(ol), ctypes.byref(osc),
                                                 _ptr(work), _stream(stream)), "ckks_encrypted_forward_host")
        return ol.value, osc.value


class ForwardGraph:
    """ckks_forward_graph_create / ckks_graph_launch: the forward's launch sequence as one CUDA graph."""

    def __init__(self, model, ct, out=None, work=None, stream=None):
        ctx = model.ctx
        self.model, self.ct = model, ct
        self.out = out if out is not None else ctx.empty_ct(ct.batch, model.final_level)
        self.work = work if work is not None else ctx.torch.empty(model.work_bytes(ct.batch),
                                                                  dtype=ctx.torch.uint8, device=ctx.device)
        i, o = ct.c(), self.out.c()
        h = ctypes.c_void_p()
        _check(lib().ckks_forward_graph_create(ctx.h, model.h, ctypes.byref(i), ctypes.byref(o), _ptr(self.work),
                                               _stream(stream), ctypes.byref(h)), "ckks_forward_graph_create")
        self.h = h
        self.out.level, self.out.scale = o.level, o.scale

    def launch(self, stream=None):
        _check(lib().ckks_graph_launch(self.h, _stream(stream)), "ckks_graph_launch")
        return self.out

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().ckks_graph_destroy(self.h)
            except Exception:
                pass
            self.h = None


def set_option(name, value):
    """ckks_set_option: process-wide kernel selection for A/B runs ("mac_tc": integer tensor-core BSGS MAC)."""
    _check(lib().ckks_set_option(name.encode(), int(value)), "ckks_set_option")


def get_option(name):
    v = _I64()
    _check(lib().ckks_get_option(name.encode(), ctypes.byref(v)), "ckks_get_option")
    return v.value


def bsgs_plan(rows, cols, x=0):
    """(t, t1, t2) of a rows x cols dense layer; x extra baby-step doublings (R5 / R5b)."""
    t, t1, t2 = _U32(), _U32(), _U32()
    _check(lib().ckks_bsgs_plan_x(int(rows), int(cols), int(x), ctypes.byref(t), ctypes.byref(t1),
                                  ctypes.byref(t2)), "ckks_bsgs_plan_x")
    return t.value, t1.value, t2.value


def model_steps(shapes, x=0):
    """Rotation steps a forward over these layer shapes needs (ckks_model_steps, R5/R5b)."""
    k = len(shapes)
    rows = (_U32 * k)(*[int(r) for r, _ in shapes])
    cols = (_U32 * k)(*[int(c) for _, c in shapes])
    ns = _U32(0)
    _check(lib().ckks_model_steps(k, rows, cols, int(x), None, ctypes.byref(ns)), "ckks_model_steps")
    st = (_I * max(1, ns.value))()
    _check(lib().ckks_model_steps(k, rows, cols, int(x), st, ctypes.byref(ns)), "ckks_model_steps")
    return list(st[: ns.value])


# C-ABI names re-exported for symmetry with include/ckks.h
def _export_names():
    g = globals()
    for name in SIGNATURES:
        g[name] = (lambda n: (lambda *a: getattr(lib(), n)(*a)))(name)


_export_names()

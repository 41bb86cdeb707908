"""CPU checks of the C-ABI boundary: the library builds/loads, exports every symbol include/ckks.h
declares, does host-side parameter validation, and refuses to compute without a GPU (no fallback).
Also checks the oracle / product separation rules (no imports either way)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2205_11935_b200 import build
    build.build()
    from paper_2205_11935_b200 import ckks
    return ckks


def header_functions():
    src = open(os.path.join(ROOT, "include", "ckks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ckks_[a-z0-9_]+)\s*\(", src)))


def test_every_header_symbol_is_exported(L):
    names = header_functions()
    assert len(names) >= 25
    out = subprocess.check_output(["nm", "-D", "--defined-only", L.lib_path()]).decode()
    exported = set(re.findall(r" T (ckks_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # and the binding declares a signature for each one
    assert set(names) <= set(L.SIGNATURES), set(names) - set(L.SIGNATURES)
    lib = L.lib()
    for n in names:
        assert getattr(lib, n) is not None


def _params(L, log_n=14, data=(60,) + (40,) * 7, special=(60,), steps=(1, 2), max_batch=4):
    bits = (ctypes.c_uint32 * (len(data) + len(special)))(*data, *special)
    st = (ctypes.c_int32 * len(steps))(*steps)
    p = L.ckks_params(log_n, len(data), len(special), bits, 3.2, 1, st, len(steps), 1, max_batch)
    return p, (bits, st)


def test_ctx_sizes_host_side(L):
    p, keep = _params(L)
    tb, kb, wb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    assert L.lib().ckks_ctx_sizes(ctypes.byref(p), ctypes.byref(tb), ctypes.byref(kb), ctypes.byref(wb)) == 0
    n, Ld = 1 << 14, 8
    key = Ld * 2 * (Ld + 1) * n * 8
    # s + pk + (relin + 2 Galois keys) + their sigma_{g^-1}-permuted copies (hoisted rotations)
    assert kb.value >= 6 * key and kb.value < 6 * key + 10 * 2 * Ld * n * 8
    assert tb.value >= 9 * 4 * n * 8
    bad, keep2 = _params(L, log_n=15)
    assert L.lib().ckks_ctx_sizes(ctypes.byref(bad), ctypes.byref(tb), ctypes.byref(kb), ctypes.byref(wb)) == L.E_PARAM
    bad, keep3 = _params(L, special=(), steps=(1,))
    assert L.lib().ckks_ctx_sizes(ctypes.byref(bad), ctypes.byref(tb), ctypes.byref(kb), ctypes.byref(wb)) == L.E_PARAM
    assert b"special" in L.lib().ckks_last_error()


def test_no_cpu_fallback(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p, keep = _params(L)
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(1024)
    st = L.lib().ckks_ctx_create(ctypes.byref(p), buf, buf, buf, None, ctypes.byref(h))
    assert st == L.E_CUDA and not h.value


def _imports(path):
    txt = open(path).read()
    return re.findall(r"^\s*(?:from|import)\s+([\w\.]+)", txt, flags=re.M)


def test_oracle_and_product_are_separate():
    prod = os.path.join(ROOT, "paper_2205_11935_b200")
    for dp, _, files in os.walk(prod):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in " ".join(_imports(os.path.join(dp, f))) if f.endswith(".py") else True
                assert "ckks_oracle" not in txt and "or_ctx" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            assert not any(m.startswith("paper_2205_11935_b200") for m in _imports(os.path.join(ROOT, "oracle", f)))
        if f.endswith(".c"):
            assert "ckks.h" not in open(os.path.join(ROOT, "oracle", f)).read()


def test_kernel_options_round_trip():
    """ckks_set_option / ckks_get_option (host-side state, no launch): every documented option reads back what
    was set, defaults are the documented ones, unknown names and out-of-range values are CKKS_E_PARAM."""
    from paper_2205_11935_b200 import ckks as G
    defaults = {"mac_tc": 0, "ip_v3": 1, "ntt_q": 15, "nvtx": 0, "giant_multi": 1}
    env = {"mac_tc": "CKKS_MAC_TC", "ip_v3": "CKKS_IP_V3", "ntt_q": "CKKS_NTT_Q", "nvtx": "CKKS_NVTX",
           "giant_multi": "CKKS_GIANT_MULTI"}
    for name, d in defaults.items():
        if env[name] not in os.environ:                         # an env override changes the default
            assert G.get_option(name) == d, name
    for name, vals in {"mac_tc": (1, 0), "ip_v3": (0, 1), "ntt_q": (0, 15, 79, 7), "nvtx": (1, 0), "giant_multi": (0, 1)}.items():
        for v in vals:
            G.set_option(name, v)
            assert G.get_option(name) == v
    for name, bad in (("mac_tc", 2), ("ip_v3", -1), ("ntt_q", 256), ("nvtx", 5), ("giant_multi", 2), ("no_such_option", 0)):
        with pytest.raises(Exception):
            G.set_option(name, bad)
    with pytest.raises(Exception):
        G.get_option("no_such_option")
    for name, d in defaults.items():
        if env[name] not in os.environ:
            G.set_option(name, d)

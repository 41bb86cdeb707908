"""fp64 CKKS encode/decode and big-integer CRT (TEST INFRASTRUCTURE ONLY).

Slots and the canonical embedding (R3, R4; "encrypt a vector of floating point numbers
into only one ciphertext"; "scale the input floating point numbers by a scale Delta, round"):
  * n = N/2 slots; slot i <-> the root zeta^{5^i mod 2N}, zeta = exp(i pi / N).
  * encode(z, Delta):  m_k = round_half_away( Delta * (2/N) * Re sum_{i<n} z_i zeta^{-k 5^i} )
    computed as Re(FFT_{2N}(Z))[k] / N, Z[5^i] = Delta z_i, Z[-5^i] = conj(Delta z_i)  (numpy FFT).
  * decode(m, Delta):  z_i = Delta^{-1} sum_k m~_k zeta^{k 5^i}, m~ the centered CRT lift mod Q_l.
A plain O(N n) evaluation of the same sums (encode_direct / decode_direct) is kept for the pins.
"""
from __future__ import annotations

import numpy as np


def slot_exponents(n_ring: int) -> np.ndarray:
    """5^i mod 2N for i < N/2 (R3)."""
    two_n = 2 * n_ring
    e = np.empty(n_ring // 2, dtype=np.int64)
    v = 1
    for i in range(n_ring // 2):
        e[i] = v
        v = (v * 5) % two_n
    return e


def round_half_away(x: np.ndarray) -> np.ndarray:
    """Round half away from zero (R16; not numpy's banker's rounding)."""
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def encode(values, scale: float, n_ring: int) -> np.ndarray:
    """Real slot vector (length <= N/2, zero-padded) -> int64 coefficients m_0..m_{N-1}."""
    z = np.zeros(n_ring // 2, dtype=np.complex128)
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size > n_ring // 2:
        raise ValueError("more values than slots")
    z[: v.size] = v
    e = slot_exponents(n_ring)
    Z = np.zeros(2 * n_ring, dtype=np.complex128)
    Z[e] = scale * z
    Z[(2 * n_ring - e) % (2 * n_ring)] = np.conj(scale * z)
    m = np.fft.fft(Z)[:n_ring].real / n_ring
    r = round_half_away(m)
    if np.max(np.abs(r), initial=0.0) >= 2.0 ** 62:
        raise OverflowError("encoded coefficient exceeds 2^62")
    return r.astype(np.int64)


def encode_const(c: float, scale: float, n_ring: int) -> np.ndarray:
    """A constant in every slot encodes exactly to round(c * scale) at coefficient 0 (R4)."""
    m = np.zeros(n_ring, dtype=np.int64)
    m[0] = int(round_half_away(np.array([c * scale]))[0])
    return m


def encode_direct(values, scale: float, n_ring: int) -> np.ndarray:
    """O(N n) definition of encode, for small-N pins only (no rounding applied)."""
    n = n_ring // 2
    z = np.zeros(n, dtype=np.complex128)
    v = np.asarray(values, dtype=np.float64).ravel()
    z[: v.size] = v
    e = slot_exponents(n_ring)
    k = np.arange(n_ring)
    zeta = np.exp(1j * np.pi / n_ring)
    M = zeta ** (-np.outer(k, e))   # [N][n]
    return scale * (2.0 / n_ring) * (M @ z).real


def crt_lift_centered(residues: np.ndarray, primes) -> list:
    """Centered CRT lift of [l+1][N] residues to Python ints in (-Q/2, Q/2]."""
    primes = [int(q) for q in primes[: residues.shape[0]]]
    Q = 1
    for q in primes:
        Q *= q
    acc = np.zeros(residues.shape[1], dtype=object)
    for i, q in enumerate(primes):
        Qi = Q // q
        ci = pow(Qi % q, -1, q)
        r = residues[i].astype(object)
        acc = acc + ((r * ci) % q) * Qi
    acc = acc % Q
    half = Q // 2
    return [int(x) - Q if int(x) > half else int(x) for x in acc]


def decode_coeffs(m_int, scale: float, n_ring: int) -> np.ndarray:
    """Integer (or float) coefficients -> complex slot values / scale, via inverse FFT."""
    m = np.array([float(x) for x in m_int], dtype=np.float64)
    M = np.zeros(2 * n_ring, dtype=np.complex128)
    M[:n_ring] = m
    ev = np.fft.ifft(M) * (2 * n_ring)     # ev[e] = sum_k m_k exp(2 pi i e k / 2N) = m(zeta^e)
    return ev[slot_exponents(n_ring)] / scale


def decode_direct(m_int, scale: float, n_ring: int) -> np.ndarray:
    """O(N n) definition of decode, for small-N pins only."""
    m = np.array([float(x) for x in m_int], dtype=np.float64)
    e = slot_exponents(n_ring)
    zeta = np.exp(1j * np.pi / n_ring)
    k = np.arange(n_ring)
    return (zeta ** np.outer(e, k) @ m) / scale


def decode(residues: np.ndarray, primes, scale: float, n_ring: int) -> np.ndarray:
    """Decrypted coefficient residues [l+1][N] -> real slot values."""
    return decode_coeffs(crt_lift_centered(residues, primes), scale, n_ring).real

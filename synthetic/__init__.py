"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no NTT, no encoding, no key switching, no
prime search).  It only:
  * names the five BASELINE.json configurations (shapes, bit sizes, seeds), and
  * draws the seeded inputs those configurations specify (fp64 vectors/matrices, and uniform
    residues in [0, q) for caller-supplied moduli q).
Both the oracle tests and the CUDA path read their inputs from here, so the two sides see
the same numbers; neither side's arithmetic lives here.

Input recipe: numpy PCG64 seeded per (config seed, purpose).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    log_n: int
    data_bits: tuple            # bit sizes of the data primes q_0..q_{L-1}
    special_bits: tuple         # () or (b,) for the special prime P
    log2_scale: float
    sigma: float = 3.2
    key_seed: int = 0x5EED0001
    enc_seed: int = 0x5EED0002
    data_seed: int = 0x5EED0003
    # workload shape
    layers: tuple = ()          # ((rows, cols), ...) dense layers, in order
    activation: str = "none"    # "none" | "square" | "cubic"
    batch: int = 1
    in_dim: int = 0
    rot_steps: tuple = ()       # for the rotation/key-switch batch (cfg3)
    note: str = ""
    weight_std: tuple = ()      # per-layer N(0, std^2)
    bias_range: float = 0.1     # U[-bias_range, bias_range]
    digits: tuple = ()          # key-switching digit sizes (R9b); () = one digit per data prime

    @property
    def n(self):
        return 1 << self.log_n

    @property
    def bits(self):
        return tuple(self.data_bits) + tuple(self.special_bits)


# BASELINE.json configs[0..4].  Readings R1, R18-R21 fix what the configs leave open.
CFG1 = Config(
    name="cfg1_tiny_dense", log_n=13, data_bits=(60, 40, 40), special_bits=(60,), log2_scale=40,
    layers=((16, 64),), activation="none", batch=1, in_dim=64, weight_std=(0.1,),
    note="N=8192, [60,40,40|60], Delta=2^40, W 16x64 ~ N(0,0.1^2), b ~ U[-0.1,0.1], x ~ U[-1,1]^64")
CFG2 = Config(
    name="cfg2_batched_ntt", log_n=14, data_bits=(50,) * 8, special_bits=(), log2_scale=40,
    batch=1024, note="1024 x 8 limbs x N=16384 uniform residues, forward then inverse NTT")
CFG3 = Config(
    name="cfg3_rotation_batch", log_n=14, data_bits=(60,) + (40,) * 7, special_bits=(60,),
    log2_scale=40, batch=256, rot_steps=(1, 2, 4, 8, 16, 32, 64, 128, 256),
    note="256 cts x [2][8][16384] uniform residues, dnum=8 (one digit per prime), 9 Galois keys")
CFG4 = Config(
    name="cfg4_two_layer_forward", log_n=14, data_bits=(60,) + (40,) * 7, special_bits=(60,),
    log2_scale=40, layers=((256, 512), (128, 256)), activation="square", batch=1, in_dim=512,
    weight_std=(1.0 / np.sqrt(512), 1.0 / np.sqrt(256)),
    note="dense 512->256, square, dense 256->128; W1 ~ N(0,1/512), W2 ~ N(0,1/256) (R20)")
CFG5 = Config(
    name="cfg5_throughput_batch", log_n=14, data_bits=(60,) + (40,) * 7, special_bits=(60,),
    log2_scale=40, layers=((256, 512), (128, 256)), activation="square", batch=1024, in_dim=512,
    weight_std=(1.0 / np.sqrt(512), 1.0 / np.sqrt(256)),
    note="1024 independent cfg4 inputs, one ciphertext each, one batched launch sequence")

# SURVEY 8(f) row f-3, reading R29: the cfg4/cfg5 network with hybrid key switching -- the same 8 data
# primes [60, 40x7], two 40-bit special primes (log QP = 420 <= 438 at N = 16384) and dnum = 5 digits
# {q0}, {q1 q2}, {q3 q4}, {q5 q6}, {q7}
CFG4_HYBRID = Config(
    name="cfg4_two_layer_forward_hybrid_ks", log_n=14, data_bits=(60,) + (40,) * 7, special_bits=(40, 40),
    log2_scale=40, layers=((256, 512), (128, 256)), activation="square", batch=1, in_dim=512,
    weight_std=(1.0 / np.sqrt(512), 1.0 / np.sqrt(256)), digits=(1, 2, 2, 2, 1),
    note="cfg4 with hybrid key switching: [60, 40x7 | 40, 40], dnum = 5 (R29)")
CFG5_HYBRID = Config(
    name="cfg5_throughput_batch_hybrid_ks", log_n=14, data_bits=(60,) + (40,) * 7, special_bits=(40, 40),
    log2_scale=40, layers=((256, 512), (128, 256)), activation="square", batch=1024, in_dim=512,
    weight_std=(1.0 / np.sqrt(512), 1.0 / np.sqrt(256)), digits=(1, 2, 2, 2, 1),
    note="cfg5 with hybrid key switching: [60, 40x7 | 40, 40], dnum = 5 (R29)")

CONFIGS = {c.name: c for c in (CFG1, CFG2, CFG3, CFG4, CFG5, CFG4_HYBRID, CFG5_HYBRID)}

_PURPOSE = {"x": 1, "w": 2, "b": 3, "residues": 4}


def _rng(seed: int, purpose: str, extra: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), _PURPOSE[purpose], int(extra)]))


def dense_problem(cfg: Config, batch: int | None = None, seed: int | None = None):
    """x ~ U[-1,1]^(batch x in_dim); per layer W ~ N(0, std^2) (rows x cols), b ~ U[-r, r]^rows."""
    seed = cfg.data_seed if seed is None else seed
    batch = cfg.batch if batch is None else batch
    x = _rng(seed, "x").uniform(-1.0, 1.0, size=(batch, cfg.in_dim))
    Ws, bs = [], []
    for li, (rows, cols) in enumerate(cfg.layers):
        Ws.append(_rng(seed, "w", li).normal(0.0, cfg.weight_std[li], size=(rows, cols)))
        bs.append(_rng(seed, "b", li).uniform(-cfg.bias_range, cfg.bias_range, size=rows))
    return {"x": x, "W": Ws, "b": bs}


def uniform_residues(seed: int, moduli, shape_prefix, n: int, tag: int = 0) -> np.ndarray:
    """Array of shape (*shape_prefix, len(moduli), n), entry [..., i, k] uniform in [0, moduli[i])."""
    g = _rng(seed, "residues", tag)
    moduli = [int(q) for q in moduli]
    out = np.empty(tuple(shape_prefix) + (len(moduli), n), dtype=np.uint64)
    for i, q in enumerate(moduli):
        out[..., i, :] = g.integers(0, q, size=tuple(shape_prefix) + (n,), dtype=np.uint64)
    return out


# NEXT f-2: the paper's frozen stack at its Table 2 presets.  Synthetic weights
# (the trained CryptoTL weights are not available); shapes are the paper's.
P2_STACK = Config(
    name="paper_p2_frozen_stack", log_n=14, data_bits=(60,) + (50,) * 6, special_bits=(60,), log2_scale=50,
    batch=128, in_dim=768,
    note="conv1d f=9 -> dense 768 + ReLU_approx -> avgpool 3 -> dense 766; N=16384, log q = 420, "
         "log Delta = 50, p = 5 items per ciphertext (Table 2 p2)")
P1_STACK = Config(
    name="paper_p1_frozen_stack", log_n=13, data_bits=(40,) + (22,) * 6, special_bits=(46,), log2_scale=22,
    batch=128, in_dim=768,
    note="Table 2 p1 chain [40, 22x6 | 46] (log q = 218), N=8192, p = 2")


def frozen_stack_weights(t: int = 768, seed: int = 0x5EED0004, f_conv: int = 9, f_pool: int = 3):
    """conv w ~ N(0, 0.3^2), W1 ~ N(0, 1/t), W2 ~ N(0, 1/(t - f_pool + 1)), biases U[-0.1, 0.1]."""
    tp = t - f_pool + 1
    return {"conv_w": _rng(seed, "w", 10).normal(0, 0.3, f_conv), "conv_b": 0.01,
            "W1": _rng(seed, "w", 11).normal(0, 1 / np.sqrt(t), (t, t)),
            "b1": _rng(seed, "b", 11).uniform(-0.1, 0.1, t),
            "W2": _rng(seed, "w", 12).normal(0, 1 / np.sqrt(tp), (tp, tp)),
            "b2": _rng(seed, "b", 12).uniform(-0.1, 0.1, tp), "f_pool": f_pool}


def frozen_stack_items(count: int, t: int = 768, seed: int = 0x5EED0005) -> np.ndarray:
    return _rng(seed, "x", 20).uniform(-1.0, 1.0, size=(count, t))

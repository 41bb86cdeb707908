"""Encrypted circuits of the frozen layers, oracle side (TEST INFRASTRUCTURE ONLY).

Follows, in the paper's order and notation:
  * Dense layer, BSGS diagonal method, Eq. 1:
        M x = sum_{k<t2} rot_{k t1}( sum_{j<t1} diag'_{k t1 + j}(M) o rot_j(x) ),
        diag'_i(M) = rot_{-floor(i/t1) t1}(diag_i(M)),  t = t1 t2,  zero-padded to t x t.
    Input packed duplicated [x || x] ("twice the number of neurons").  Readings R4-R8.
  * Square activation (BASELINE.json cfg4) and the cubic ReLU approximation, Eq. 2:
        ReLU_approx(z) = -0.0061728 z^3 + 0.092593 z^2 + 0.59259 z + 0.49383   (schedule R23).
  * Replicate y + rot_{-t}(y) restoring the duplicated layout (R-replicate).
  * The float64 plaintext reference forward these must match after decryption (north_star, 1e-3).
Ring arithmetic is the C oracle's (`Context`); nothing here touches residues except through it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import encoding

RELU_APPROX = (-0.0061728, 0.092593, 0.59259, 0.49383)   # c3, c2, c1, c0  (Eq. 2)


@dataclass
class Ct:
    data: np.ndarray      # [2 (or 3)][level+1][N] NTT-domain residues
    scale: float

    @property
    def level(self):
        return self.data.shape[1] - 1


def bsgs_split(rows: int, cols: int, x: int = 0):
    """t = max(rows, cols) (P:L96 zero padding); t1 = 2^ceil(ceil(log2 t)/2); t padded to t1 | t (R5).
    x > 0: t1 = 2^min(lg, ceil(lg/2) + x) (R5b, more baby steps; the same Eq. 1 product)."""
    t = max(rows, cols)
    lg = max(0, math.ceil(math.log2(t)))
    t1 = 1 << min(lg, math.ceil(lg / 2) + x)
    t = -(-t // t1) * t1
    return t, t1, t // t1


def diagonals(W: np.ndarray, x: int = 0):
    """diag_i(M)[s] = Mpad[s][(s + i) mod t]  for i < t."""
    rows, cols = W.shape
    t, t1, t2 = bsgs_split(rows, cols, x)
    Mp = np.zeros((t, t))
    Mp[:rows, :cols] = W
    s = np.arange(t)
    return np.stack([Mp[s, (s + i) % t] for i in range(t)]), (t, t1, t2)


def diag_prime_slots(W: np.ndarray, n_slots: int, x: int = 0):
    """diag'_{k t1 + j} = rot_{-k t1}(diag_{k t1 + j}) as full slot vectors (zero-filled, R4)."""
    D, (t, t1, t2) = diagonals(W, x)
    if 2 * t > n_slots:
        raise ValueError("2t exceeds the slot count")
    out = np.zeros((t, n_slots))
    for i in range(t):
        k = i // t1
        out[i, k * t1: k * t1 + t] = D[i]
    return out, (t, t1, t2)


@dataclass
class EncodedLayer:
    """Shared encoded plaintexts of one dense layer (integer coefficients, R8)."""
    rows: int
    cols: int
    t: int
    t1: int
    t2: int
    level: int                  # level of the input ciphertext
    pt_scale: float             # Delta_w = q_level (R8)
    bias_scale: float           # = input scale (exact after rescale)
    diag_coeffs: np.ndarray     # [t][N] int64
    bias_coeffs: np.ndarray     # [N] int64


def encode_layer(ctx, W, b, level: int, in_scale: float, x: int = 0) -> EncodedLayer:
    W = np.asarray(W, dtype=np.float64)
    rows, cols = W.shape
    slots, (t, t1, t2) = diag_prime_slots(W, ctx.n // 2, x)
    q_l = float(ctx.primes[level])
    coeffs = np.stack([encoding.encode(slots[i], q_l, ctx.n) for i in range(t)])
    bias = np.zeros(ctx.n // 2)
    if b is not None:
        bias[:rows] = b
    bcoef = encoding.encode(bias, in_scale, ctx.n)
    return EncodedLayer(rows, cols, t, t1, t2, level, q_l, in_scale, coeffs, bcoef)


def rotation_steps_for(layers_shapes, x: int = 0):
    """Every Galois step the forward needs: baby 1..t1-1, giant k t1, replicate -t (R5)."""
    steps = set()
    for li, (rows, cols) in enumerate(layers_shapes):
        t, t1, t2 = bsgs_split(rows, cols, x)
        steps.update(range(1, t1))
        steps.update(k * t1 for k in range(1, t2))
        if li > 0:
            steps.add(-t)
    return sorted(steps)


class OpCount:
    def __init__(self):
        self.rot = 0
        self.mul_plain = 0
        self.add = 0


def _bsgs_sum(ctx, ct_data, level, t1, t2, giant, baby_steps, pt_coeffs, hoisted, ops):
    """sum_k rot_{k giant}(sum_j pt_{k t1 + j} o rot_{baby_j}(x))  (Eq. 1), in the order of Eq. 1.
    hoisted = 0: every rotation non-hoisted (R11); 1: baby steps hoisted (R11b); 2: double hoisting
    (R11c) -- baby steps, inner sums and giant steps in the Q_l P basis, one ModDown at the end."""
    l = level
    if hoisted == 2:
        baby = [ctx.lift_qp(ct_data) if s == 0 else ctx.rotate_hoisted_qp(ct_data, s) for s in baby_steps]
        plain, mul, add, rot = ctx.plain_qp, ctx.mul_plain_qp, ctx.add_qp, ctx.rotate_qp
    else:
        r = ctx.rotate_hoisted if hoisted else ctx.rotate
        baby = [ct_data if s == 0 else r(ct_data, s) for s in baby_steps]
        plain, mul, add, rot = ctx.plain, ctx.mul_plain, ctx.add, ctx.rotate
    if ops:
        ops.rot += sum(1 for s in baby_steps if s != 0)
    y = None
    for k in range(t2):
        w = None
        for j in range(t1):
            term = mul(baby[j], plain(pt_coeffs[k * t1 + j], l))
            w = term if w is None else add(w, term)
            if ops:
                ops.mul_plain += 1
        if k > 0:
            w = rot(w, k * giant)
            if ops:
                ops.rot += 1
        y = w if y is None else add(y, w)
    return ctx.moddown(y) if hoisted == 2 else y


def matvec(ctx, ct: Ct, layer: EncodedLayer, ops: OpCount | None = None, hoisted: int = 0) -> Ct:
    """Eq. 1 then one rescale (R7) then + bias (R-bias).  t1+t2-2 rotations, t pt-ct mults.
    hoisted=1: the t1-1 baby-step rotations are hoisted (NEXT f-1, R11b); 2: double hoisting (R11c)."""
    l = ct.level
    assert layer.level == l, "layer encoded for another level"
    y = _bsgs_sum(ctx, ct.data, l, layer.t1, layer.t2, layer.t1, list(range(layer.t1)), layer.diag_coeffs,
                  int(hoisted), ops)
    y = ctx.rescale(y)
    out_scale = ct.scale * layer.pt_scale / float(ctx.primes[l])
    y = ctx.add_plain(y, ctx.plain(layer.bias_coeffs, l - 1))
    return Ct(y, out_scale)


def square(ctx, z: Ct) -> Ct:
    """rescale(relin(z (x) z)): depth 1 (BASELINE cfg4 activation)."""
    l = z.level
    y = ctx.rescale(ctx.relinearize(ctx.tensor(z.data, z.data)))
    return Ct(y, z.scale * z.scale / float(ctx.primes[l]))


def cubic_c0_coeffs(c0: float, valid: int, scale: float, n: int) -> np.ndarray:
    """The constant term restricted to the valid slots [0, valid) (R23: keeps the zero padding the
    following replicate relies on), encoded at the activation output scale."""
    v = np.zeros(n // 2)
    v[:valid] = c0
    return encoding.encode(v, scale, n)


def cubic(ctx, z: Ct, coeffs=RELU_APPROX, valid: int | None = None, c0_coeffs=None) -> Ct:
    """Eq. 2 at depth 2, schedule R23:
       z2 = rescale(relin(z (x) z));  a = rescale(z o [c3]_{q_l}) + [c2]_S;
       h = rescale(relin(z2 (x) a));  g = drop(rescale(z o [c1]_{S3 q_l / S})) + [c0]_{S3};  out = h + g.
    [c0]_{S3} is the constant in every slot (valid=None) or c0 on slots [0, valid) only."""
    c3, c2, c1, c0 = coeffs
    l = z.level
    S = z.scale
    ql, ql1 = float(ctx.primes[l]), float(ctx.primes[l - 1])
    n = ctx.n
    z2 = ctx.rescale(ctx.relinearize(ctx.tensor(z.data, z.data)))               # l-1, S^2/ql
    a = ctx.rescale(ctx.mul_plain(z.data, ctx.plain(encoding.encode_const(c3, ql, n), l)))
    a = ctx.add_plain(a, ctx.plain(encoding.encode_const(c2, S, n), l - 1))     # l-1, S
    h = ctx.rescale(ctx.relinearize(ctx.tensor(z2, a)))                         # l-2, S3
    S3 = (S * S / ql) * S / ql1
    g = ctx.rescale(ctx.mul_plain(z.data, ctx.plain(encoding.encode_const(c1, S3 * ql / S, n), l)))
    g = ctx.drop_level(g, l - 2)
    if c0_coeffs is None:
        c0_coeffs = encoding.encode_const(c0, S3, n) if valid is None else cubic_c0_coeffs(c0, valid, S3, n)
    g = ctx.add_plain(g, ctx.plain(c0_coeffs, l - 2))
    return Ct(ctx.add(h, g), S3)


def replicate(ctx, y: Ct, t: int) -> Ct:
    """y + rot_{-t}(y): [y | 0] -> [y | y] on slots [0, 2t) (P:L116 duplicated layout)."""
    return Ct(ctx.add(y.data, ctx.rotate(y.data, -t)), y.scale)


def activation_plaintexts(ctx, layers, activation: str):
    """Masked constant-term plaintexts of the cubic activations (one per non-final layer), R23."""
    if activation != "cubic":
        return None
    out = []
    for lay in layers[:-1]:
        S = lay.bias_scale                          # dense output scale = its input scale (R8)
        l = lay.level - 1
        ql, ql1 = float(ctx.primes[l]), float(ctx.primes[l - 1])
        S3 = (S * S / ql) * S / ql1
        out.append(cubic_c0_coeffs(RELU_APPROX[3], lay.rows, S3, ctx.n))
    return np.stack(out)


def forward(ctx, ct: Ct, layers, activation: str = "square", ops: OpCount | None = None,
            hoisted: bool = False) -> Ct:
    """dense_1 -> act -> replicate -> dense_2 -> ... (P:L118 frozen stack, BASELINE cfg4)."""
    for li, layer in enumerate(layers):
        if li > 0:
            ct = replicate(ctx, ct, layer.t)
            if ops:
                ops.rot += 1
        ct = matvec(ctx, ct, layer, ops, hoisted=hoisted)
        if li < len(layers) - 1:
            if activation == "square":
                ct = square(ctx, ct)
            elif activation == "cubic":
                ct = cubic(ctx, ct, valid=layer.rows)
            elif activation != "none":
                raise ValueError(activation)
    return ct


def encode_model(ctx, Ws, bs, level: int, scale: float, activation: str, x: int = 0):
    """Encode every layer at the level/scale its input will have (R8 scale bookkeeping)."""
    layers = []
    s = scale
    l = level
    for li, (W, b) in enumerate(zip(Ws, bs)):
        lay = encode_layer(ctx, W, b, l, s, x)
        layers.append(lay)
        l -= 1                                   # one rescale in the dense layer; scale unchanged
        if li < len(Ws) - 1:
            if activation == "square":
                s = s * s / float(ctx.primes[l])
                l -= 1
            elif activation == "cubic":
                ql, ql1 = float(ctx.primes[l]), float(ctx.primes[l - 1])
                s = (s * s / ql) * s / ql1
                l -= 2
    return layers


def plain_forward(x, Ws, bs, activation: str = "square"):
    """float64 reference (north_star): y1 = W1 x + b1; z = act(y1); y = W2 z + b2 ..."""
    y = np.asarray(x, dtype=np.float64)
    for li, (W, b) in enumerate(zip(Ws, bs)):
        y = W @ y + b
        if li < len(Ws) - 1:
            if activation == "square":
                y = y * y
            elif activation == "cubic":
                c3, c2, c1, c0 = RELU_APPROX
                y = ((c3 * y + c2) * y + c1) * y + c0
    return y


def pack_input(x, t: int, n_slots: int) -> np.ndarray:
    """[x || x] on slots [0, 2t), zeros elsewhere."""
    v = np.zeros(n_slots)
    x = np.asarray(x, dtype=np.float64)
    v[: x.size] = x
    v[t: t + x.size] = x
    return v


# =============================================================================== NEXT f-2: frozen stack
# The paper's frozen server stack: Conv1D (f=9) -> Dense 768 + ReLU_approx (Eq. 2)
# -> AvgPool (f=3) -> [Dropout = identity at inference] -> Dense 766, depth 6, with p items per
# ciphertext.  Readings R25-R28:
#   R25 packing: p = floor(n / (2t + c)) items (c = conv half-width, 0 without conv; = the paper's
#       floor(#slots / 2 #neurons) when c is small enough), region size R = floor(n / p); item r at
#       slots [rR, rR + t), zeros in [rR + t, (r+1)R) until a replicate duplicates it.
#   R26 conv1d ('same', zero padded, P:L98 packed SISO): out[k] = sum_{i<f} w_i x[k + i - c] + b,
#       = sum_i m_i o rot_{i-c}(x), m_i = w_i on every item's [rR, rR + t); f mults, f-1 rotations.
#   R27 avgpool (x_o = (1/f) sum_i rot_{-i}(x)): out[k] = (1/f) sum_{i<f} x[k - i],
#       valid on [f-1, t) of each item (the 1/f plaintext is the validity mask); f-1 rotations, 1 mult.
#   R28 the dense after the pool reads its input from slots [f-1, t): cols = t, columns < f-1 zero.

def packing(n_slots: int, t: int, conv_half: int = 0):
    """(p, R): items per ciphertext and region size (R25)."""
    p = n_slots // (2 * t + conv_half)
    if p < 1:
        raise ValueError("item does not fit")
    return p, n_slots // p


def region_mask(values, t: int, region: int, items: int, n_slots: int, offset: int = 0) -> np.ndarray:
    """Per-slot vector holding `values` (length <= t, or a scalar) at [rR + offset, ...) for every item."""
    out = np.zeros(n_slots)
    v = np.broadcast_to(np.asarray(values, dtype=np.float64), (t - offset,)) if np.ndim(values) == 0 \
        else np.asarray(values, dtype=np.float64)
    for r in range(items):
        out[r * region + offset: r * region + offset + v.size] = v
    return out


@dataclass
class HoistedLayer:
    """A linear layer evaluated as  y = sum_k rot_{k g}( sum_j pt_{k,j} o rot_{s_j}(x) )  (+ bias), with
    baby steps s_0 = 0, s_1.. and (for the BSGS dense) giant step g = t1.  Shared encodings (R8)."""
    kind: str                   # "dense" | "conv" | "pool"
    t: int
    t2: int
    baby_steps: list
    giant: int
    level: int
    pt_scale: float
    bias_scale: float
    pt_coeffs: np.ndarray       # [t2 * t1][N] int64
    bias_coeffs: np.ndarray     # [N] int64 or None
    rows: int = 0
    cols: int = 0

    @property
    def t1(self):
        return len(self.baby_steps)


def encode_dense_packed(ctx, W, b, level, in_scale, region, items) -> HoistedLayer:
    """BSGS dense (Eq. 1) with diag' replicated in every item region."""
    W = np.asarray(W, dtype=np.float64)
    rows, cols = W.shape
    D, (t, t1, t2) = diagonals(W)
    n = ctx.n // 2
    q_l = float(ctx.primes[level])
    pts = []
    for i in range(t):
        k = i // t1
        v = np.zeros(n)
        for r in range(items):
            v[r * region + k * t1: r * region + k * t1 + t] = D[i]
        pts.append(encoding.encode(v, q_l, ctx.n))
    bias = None
    if b is not None:
        bias = encoding.encode(region_mask(np.asarray(b), t, region, items, n), in_scale, ctx.n)
    return HoistedLayer("dense", t, t2, list(range(t1)), t1, level, q_l, in_scale, np.stack(pts), bias, rows, cols)


def encode_conv(ctx, w, bias, t, level, in_scale, region, items) -> HoistedLayer:
    """R26: taps ordered so that step 0 (the centre tap) comes first."""
    w = np.asarray(w, dtype=np.float64)
    f = w.size
    c = (f - 1) // 2
    order = [c] + [i for i in range(f) if i != c]
    n = ctx.n // 2
    q_l = float(ctx.primes[level])
    pts = np.stack([encoding.encode(region_mask(w[i], t, region, items, n), q_l, ctx.n) for i in order])
    bc = None
    if bias is not None:
        bc = encoding.encode(region_mask(float(bias), t, region, items, n), in_scale, ctx.n)
    return HoistedLayer("conv", t, 1, [i - c for i in order], 0, level, q_l, in_scale, pts, bc, t, t)


def encode_pool(ctx, f, t, level, region, items) -> HoistedLayer:
    """R27: f copies of the 1/f validity mask on [f-1, t); steps 0, -1, .., -(f-1)."""
    n = ctx.n // 2
    q_l = float(ctx.primes[level])
    m = encoding.encode(region_mask(1.0 / f, t, region, items, n, offset=f - 1), q_l, ctx.n)
    return HoistedLayer("pool", t, 1, [-i for i in range(f)], 0, level, q_l, 0.0, np.stack([m] * f), None, t, t)


def apply_layer(ctx, ct: Ct, lay: HoistedLayer, hoisted: int = 1, ops: OpCount | None = None) -> Ct:
    """y = sum_k rot_{k g}(sum_j pt_{k,j} o rot_{s_j}(x)), one rescale, + bias (Eq. 1 / R26 / R27)."""
    l = ct.level
    assert lay.level == l
    y = _bsgs_sum(ctx, ct.data, l, lay.t1, lay.t2, lay.giant, lay.baby_steps, lay.pt_coeffs, int(hoisted), ops)
    y = ctx.rescale(y)
    if lay.bias_coeffs is not None:
        y = ctx.add_plain(y, ctx.plain(lay.bias_coeffs, l - 1))
    return Ct(y, ct.scale * lay.pt_scale / float(ctx.primes[l]))


def frozen_stack_params(t: int = 768, f_conv: int = 9, f_pool: int = 3):
    return {"t": t, "f_conv": f_conv, "f_pool": f_pool}


def frozen_stack_steps(t, t_dense_shapes, f_conv, f_pool):
    c = (f_conv - 1) // 2
    steps = set(d for d in range(-c, c + 1) if d != 0)
    steps.update(-i for i in range(1, f_pool))
    for rows, cols in t_dense_shapes:
        tt, t1, t2 = bsgs_split(rows, cols)
        steps.update(range(1, t1))
        steps.update(k * t1 for k in range(1, t2))
        steps.add(-tt)
    return sorted(steps)


def encode_frozen_stack(ctx, weights, level, scale, region, items):
    """weights: dict conv_w (f), conv_b, W1 (t x t), b1 (t), W2 (t-fp+1 x t-fp+1), b2; returns the
    stage list [(layer, activation, replicate_t)] with levels/scales of the depth-6 schedule."""
    t = weights["W1"].shape[1]
    fp = weights["f_pool"]
    stages = []
    l, s = level, scale
    conv = encode_conv(ctx, weights["conv_w"], weights["conv_b"], t, l, s, region, items)
    stages.append((conv, "none", 0))
    l -= 1
    d1 = encode_dense_packed(ctx, weights["W1"], weights["b1"], l, s, region, items)
    stages.append((d1, "cubic", t))
    l -= 1
    ql, ql1 = float(ctx.primes[l]), float(ctx.primes[l - 1])
    s = (s * s / ql) * s / ql1
    l -= 2
    pool = encode_pool(ctx, fp, t, l, region, items)
    stages.append((pool, "none", 0))
    l -= 1
    W2 = np.zeros((weights["W2"].shape[0], t))
    W2[:, fp - 1:] = weights["W2"]                     # R28: input slots [f-1, t)
    d2 = encode_dense_packed(ctx, W2, weights["b2"], l, s, region, items)
    stages.append((d2, "none", t))
    return stages


def cubic_masked_coeffs(ctx, rows, t, region, items, scale):
    v = region_mask(RELU_APPROX[3], t, region, items, ctx.n // 2)
    v = np.where(np.arange(ctx.n // 2) % region < rows, v, 0.0) if items else v
    return encoding.encode(v, scale, ctx.n)


def forward_stages(ctx, ct: Ct, stages, region, items, hoisted=True, ops=None) -> Ct:
    for lay, act, rep_t in stages:
        if rep_t:
            ct = replicate(ctx, ct, rep_t)
            if ops:
                ops.rot += 1
        ct = apply_layer(ctx, ct, lay, hoisted, ops)
        if act == "cubic":
            l = ct.level
            S = ct.scale
            ql, ql1 = float(ctx.primes[l]), float(ctx.primes[l - 1])
            S3 = (S * S / ql) * S / ql1
            c0 = cubic_masked_coeffs(ctx, lay.rows, lay.t, region, items, S3)
            ct = cubic(ctx, ct, c0_coeffs=c0)
        elif act == "square":
            ct = square(ctx, ct)
    return ct


def conv_same(x, w, b):
    f = len(w)
    c = (f - 1) // 2
    xp = np.concatenate([np.zeros(c), x, np.zeros(c)])
    return np.array([np.dot(w, xp[k:k + f]) for k in range(len(x))]) + b


def pool_valid_right(x, f):
    return np.array([np.mean(x[k - f + 1:k + 1]) for k in range(f - 1, len(x))])


def plain_frozen_forward(x, weights):
    """float64 twin of the frozen stack (dropout = identity at inference)."""
    y = conv_same(np.asarray(x, dtype=np.float64), weights["conv_w"], weights["conv_b"])
    y = weights["W1"] @ y + weights["b1"]
    c3, c2, c1, c0 = RELU_APPROX
    y = ((c3 * y + c2) * y + c1) * y + c0
    y = pool_valid_right(y, weights["f_pool"])
    return weights["W2"] @ y + weights["b2"]


def pack_items(xs, t, region, n_slots):
    v = np.zeros(n_slots)
    for r, x in enumerate(xs):
        v[r * region: r * region + len(x)] = x
    return v

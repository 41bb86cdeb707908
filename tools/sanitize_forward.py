"""One small double-hoisted forward through the C-ABI for compute-sanitizer (racecheck / synccheck /
memcheck): N=4096, [60, 40x5 | 60], layers 64x128 -> square -> 32x64, t1 = 64 / 32 (x = 1), B = 33 in
one launch sequence (max_batch = 33), so k_ks_ip_mma2 and k_bsgs_mac_mma run 3 batch tiles (16 + 16 + 1)
through their cp.async rings, k_ks_ip_giant its unroll-4 body and remainder, and k_ks_modup both ModUp
forms.  Library encoders only (no oracle): the sanitizer checks memory/synchronisation, not values."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402


def main():
    import torch
    B = int(os.environ.get("SAN_B", "33"))
    cfg = S.Config(name="san", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(60,), log2_scale=40,
                   layers=((64, 128), (32, 64)), activation="square", in_dim=128,
                   weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64)))
    x = 1
    steps = G.model_steps(cfg.layers, x)
    g = G.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, key_seed=3, rot_steps=steps, max_batch=B,
                  bsgs_baby_extra=x)
    D = 2.0 ** 40
    levels, scales, _ = g.model_plan(cfg.layers, G.ACT_SQUARE, g.top_level, D)
    prob = S.dense_problem(cfg, batch=B)
    layers = [G.Layer(g, r, c, levels[i], W=prob["W"][i], bias=prob["b"][i], in_scale=scales[i])
              for i, (r, c) in enumerate(cfg.layers)]
    model = G.Model(g, layers, G.ACT_SQUARE)
    model.set_hoisting(int(os.environ.get("SAN_HOIST", "2")))
    t0 = G.bsgs_plan(*cfg.layers[0], x)[0]
    ms = []
    for b in range(B):
        v = np.zeros(g.n // 2)
        v[:128] = prob["x"][b]
        v[t0:t0 + 128] = prob["x"][b]
        ms.append(g.encode(v, D))
    ct = g.encrypt(np.stack(ms), 5, 0, D)
    out = model.forward(ct)
    torch.cuda.synchronize()
    y = g.decode(G.u64_view(g.decrypt(out))[0], out.level, out.scale, 32)
    ref = prob["W"][1] @ (prob["W"][0] @ prob["x"][0] + prob["b"][0]) ** 2 + prob["b"][1]
    print("sanitize_forward ok, max err", float(np.max(np.abs(y - ref))), "launches", g.launches())


if __name__ == "__main__":
    main()

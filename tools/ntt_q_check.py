"""A/B of the CTA-pair NTT schedule (ntt_c.cuh; ckks_set_option("ntt_q", mask): 0 whole-limb kernels, 3 cluster
schedule with TMA row copies, 67 the same with plain 256-bit accesses) on the cfg2 batch NTT (1024 x 8 limbs,
N = 16384, 50-bit chain), a 40-bit chain and smaller rings: same bits as the whole-limb kernels, device time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2205_11935_b200 import ckks as G  # noqa: E402


def run(log_n, bits, batch, reps=20):
    dev = torch.device("cuda", 0)
    ctx = G.Context(log_n, bits, (), want_relin=False, max_batch=1, device=dev)
    x = torch.empty((batch, len(bits), ctx.n), dtype=torch.int64, device=dev)
    for i, q in enumerate(ctx.primes):
        x[:, i].random_(0, q)
    x[0, :, :64] = 0
    for i, q in enumerate(ctx.primes):
        x[1, i, :] = q - 1
    res = {}
    ref = {}
    old = G.get_option("ntt_q")
    for mask in (0, 3, 67):
        G.set_option("ntt_q", mask)
        y = x.clone()
        ctx.ntt_fwd(y)
        f = y.clone()
        ctx.ntt_inv(y)
        torch.cuda.synchronize()
        rt = bool(torch.equal(y, x))
        if mask == 0:
            ref["f"] = f
        t = {}
        for name, fn in (("fwd", ctx.ntt_fwd), ("inv", ctx.ntt_inv)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                fn(y)
            e0.record()
            for _ in range(reps):
                fn(y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            t[name] = {"ms": round(ms, 4), "GBps": round(2 * 8 * ctx.n * len(bits) * batch / ms / 1e6, 1)}
        res[f"ntt_q={mask}"] = {"round_trip": rt, "fwd_same_as_ntt_q0": bool(torch.equal(f, ref["f"])), **t}
    # mixed: forward with one schedule, inverse with the other
    G.set_option("ntt_q", 1)
    y = x.clone(); ctx.ntt_fwd(y); G.set_option("ntt_q", 0); ctx.ntt_inv(y)
    res["fwd_q_inv_old_round_trip"] = bool(torch.equal(y, x))
    G.set_option("ntt_q", 2)
    y = x.clone(); ctx.ntt_fwd(y); ctx.ntt_inv(y)
    res["fwd_old_inv_q_round_trip"] = bool(torch.equal(y, x))
    G.set_option("ntt_q", old)
    return res


if __name__ == "__main__":
    out = {"cfg2_50bit_n16384": run(14, (50,) * 8, 1024),
           "40bit_n16384": run(14, (60, 40, 40, 40, 40, 40, 40, 40), 512),
           "40bit_n8192": run(13, (40, 22, 22, 22, 46), 512),
           "n4096": run(12, (60, 40, 40, 45, 50), 256)}
    print(json.dumps(out, indent=1))

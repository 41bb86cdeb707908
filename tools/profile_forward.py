"""Profiling driver for ncu: setup outside the profiled range, then exactly one pass of the chosen
workload between cudaProfilerStart/Stop (use `ncu --profile-from-start off`).

  python tools/profile_forward.py --mode forward --batch 256     # one cfg5-style batched forward
  python tools/profile_forward.py --mode ntt                     # cfg2: one forward + one inverse NTT
  python tools/profile_forward.py --mode ks                      # cfg3: 256 cts rotated by 9 steps
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--mode", default="forward", choices=["forward", "ntt", "ks"])
    p.add_argument("--batch", type=int, default=256)
    p.add_argument("--max-batch", type=int, default=256)
    p.add_argument("--no-hoist", action="store_true")
    p.add_argument("--hoisting", type=int, default=2)
    p.add_argument("--ks", default="hybrid", choices=("hybrid", "single"))
    a = p.parse_args()
    dev = torch.device("cuda", 0)
    if a.mode == "forward":
        ctx, model, ct, _ = bench.build_forward(G, bench.workload_cfg(S, a.ks), a.batch, a.max_batch, dev,
                                                hoisted=0 if a.no_hoist else a.hoisting)
        out = ctx.empty_ct(a.batch, model.final_level)
        work = torch.empty(model.work_bytes(a.batch), dtype=torch.uint8, device=dev)
        model.forward(ct, out, work)
        torch.cuda.synchronize()
        l0 = ctx.launches()
        t0 = time.perf_counter()
        torch.cuda.profiler.start()
        model.forward(ct, out, work)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(f"forward batch={a.batch}: {ctx.launches() - l0} launches, {time.perf_counter() - t0:.3f} s")
    elif a.mode == "ntt":
        cfg = S.CFG2
        ctx = G.Context(cfg.log_n, cfg.data_bits, (), want_relin=False, max_batch=1, device=dev)
        x = torch.empty((cfg.batch, len(cfg.data_bits), ctx.n), dtype=torch.int64, device=dev)
        for i, q in enumerate(ctx.primes):
            x[:, i].random_(0, q)
        ctx.ntt_fwd(x)
        ctx.ntt_inv(x)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        ctx.ntt_fwd(x)
        ctx.ntt_inv(x)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print("ntt ok")
    else:
        cfg = S.CFG3
        ctx = G.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, key_seed=cfg.key_seed, rot_steps=cfg.rot_steps,
                        want_relin=False, max_batch=cfg.batch, device=dev)
        x = torch.empty((cfg.batch, 2, ctx.n_data, ctx.n), dtype=torch.int64, device=dev)
        for i in range(ctx.n_data):
            x[:, :, i].random_(0, ctx.primes[i])
        ct = G.Ciphertext(x, ctx.top_level, 2.0 ** 40)
        out = ctx.empty_ct(cfg.batch, ctx.top_level)
        ctx.rotate(ct, 1, out)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for st in cfg.rot_steps:
            ctx.rotate(ct, st, out)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print("ks ok")


if __name__ == "__main__":
    main()

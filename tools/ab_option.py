"""A/B of a process-wide kernel option (ckks_set_option) on one B = 256 chunk of the cfg5 forward:
same bits (checked word for word), device time per forward and per kernel (library probe).

  python tools/ab_option.py ip_v3 0 1          # baby-step IP: Karatsuba kernel vs pre-multiplied key kernel
  python tools/ab_option.py mac_tc 0 1 --ks single
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("option")
    p.add_argument("values", nargs="+", type=int)
    p.add_argument("--batch", type=int, default=256)
    p.add_argument("--reps", type=int, default=4)
    p.add_argument("--ks", default="hybrid", choices=("hybrid", "single"))
    a = p.parse_args()
    dev = torch.device("cuda", 0)
    ctx, model, ct, _ = bench.build_forward(G, bench.workload_cfg(S, a.ks), a.batch, a.batch, dev, hoisted=2)
    out = ctx.empty_ct(a.batch, model.final_level)
    work = torch.empty(model.work_bytes(a.batch), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    old = G.get_option(a.option)
    ref, res = None, {}
    try:
        for v in a.values:
            G.set_option(a.option, v)
            model.forward(ct, out, work)
            torch.cuda.synchronize()
            bits = out.data.clone()
            ref = bits if ref is None else ref
            ctx.probe(G.PROBE_ALL)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.reps):
                model.forward(ct, out, work)
            e1.record(stream)
            torch.cuda.synchronize()
            per = ctx.probe_read_all()
            ctx.probe(G.PROBE_OFF)
            ks = sorted(((k, w) for k, w in per.items() if isinstance(w, dict) and "ms" in w),
                        key=lambda kv: -kv[1]["ms"])[:6]
            res[f"{a.option}={v}"] = {"ms_per_forward_chunk": round(e0.elapsed_time(e1) / a.reps, 3),
                                      "same_bits": bool(torch.equal(bits, ref)),
                                      "kernels_ms": {k: round(w["ms"] / a.reps, 3) for k, w in ks}}
    finally:
        G.set_option(a.option, old)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

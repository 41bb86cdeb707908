"""A/B of a process-wide kernel option on the paper's p1 frozen stack (N = 8192) and the cfg1 latency line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("option")
p.add_argument("values", nargs="+", type=int)
a = p.parse_args()
args = argparse.Namespace(steps=5, no_hoist=False, hoisting=2)
dev = torch.device("cuda", 0)
old = G.get_option(a.option)
res = {}
for v in a.values:
    G.set_option(a.option, v)
    r = bench.bench_frozen_stack(G, S, dev, args, S.P1_STACK)
    lat = bench.bench_latency(G, S, dev, args)
    res[f"{a.option}={v}"] = {"p1_ms_per_batch": r["ms_per_batch"], "p1_err": r["max_abs_err_items"],
                              "cfg1_us": lat["cfg1_tiny_dense"]["us_per_forward"],
                              "cfg4_us": lat["cfg4_two_layer_forward"]["us_per_forward"]}
G.set_option(a.option, old)
print(json.dumps(res, indent=1))

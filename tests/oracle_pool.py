"""Process pool running the CPU oracle for sampled ciphertexts of a large GPU batch (test infrastructure).

The GPU parity tests of the bench's launch shapes (max_batch up to 256, batches of 100+ ciphertexts)
need the oracle's forward for many ciphertexts; one oracle forward is 0.6 s (N=4096) to 12 s (N=16384)
single-threaded, so the references are computed by a pool of worker processes.  Every worker rebuilds
the oracle context, keys and encoded layers from the same seeded spec (spawn start method: no state
is inherited from the CUDA-initialised parent) and returns the oracle output residues of the indices
it is given.  Nothing here touches the CUDA path.
"""
from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np

_W = {}


def _dense_setup(spec, keys):
    import oracle
    from oracle import circuits as OC
    from oracle import encoding as OE
    import synthetic as S
    cfg = spec["cfg"]
    x = spec.get("x", 0)
    o = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, digits=cfg.digits or None)
    if keys:
        o.keygen(cfg.key_seed, OC.rotation_steps_for(cfg.layers, x))
    prob = S.dense_problem(cfg, batch=spec["batch"])
    D = 2.0 ** cfg.log2_scale
    layers = OC.encode_model(o, prob["W"], prob["b"], o.top_level, D, spec["activation"], x)

    def message(b):
        return OE.encode(OC.pack_input(prob["x"][b], layers[0].t, o.n // 2), D, o.n)

    def forward(b):
        ref = OC.forward(o, OC.Ct(o.encrypt(message(b), cfg.enc_seed, b), D), layers, spec["activation"],
                         hoisted=spec.get("hoisting", 0))
        y = OC.plain_forward(prob["x"][b], prob["W"], prob["b"], spec["activation"])
        dec = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
        return ref.data, ref.scale, float(np.max(np.abs(dec[: y.size] - y)))

    return {"o": o, "layers": layers, "message": message, "forward": forward, "prob": prob}


def _stack_setup(spec, keys):
    import oracle
    from oracle import circuits as OC
    from oracle import encoding as OE
    import synthetic as S
    cfg = spec["cfg"]
    t = spec["t"]
    n = 1 << cfg.log_n
    p, R = OC.packing(n // 2, t, 4)
    wts = S.frozen_stack_weights(t)
    steps = OC.frozen_stack_steps(t, [(t, t), (t - 2, t)], 9, 3)
    o = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, digits=cfg.digits or None)
    if keys:
        o.keygen(cfg.key_seed, steps)
    D = 2.0 ** cfg.log2_scale
    stages = OC.encode_frozen_stack(o, wts, o.top_level, D, R, p)
    xs = S.frozen_stack_items(spec["batch"] * p, t)

    def message(b):
        return OE.encode(OC.pack_items(xs[b * p:(b + 1) * p], t, R, n // 2), D, n)

    def forward(b):
        ref = OC.forward_stages(o, OC.Ct(o.encrypt(message(b), cfg.enc_seed, b), D), stages, R, p,
                                hoisted=spec.get("hoisting", 1))
        y = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
        err = 0.0
        for r in range(p):
            ref_f = OC.plain_frozen_forward(xs[b * p + r], wts)
            err = max(err, float(np.max(np.abs(y[r * R: r * R + ref_f.size] - ref_f))))
        return ref.data, ref.scale, err

    return {"o": o, "stages": stages, "message": message, "forward": forward, "items": xs, "p": p, "R": R,
            "weights": wts}


def setup(spec, keys=True):
    """Oracle context + encodings of a spec (keys=False: the encodings and messages only, for the tests'
    own process)."""
    return _stack_setup(spec, keys) if spec["kind"] == "stack" else _dense_setup(spec, keys)


def _init(spec):
    _W["s"] = setup(spec)


def _run(b):
    data, scale, err = _W["s"]["forward"](int(b))
    return int(b), data, scale, err


def workers_for(count: int) -> int:
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return max(1, min(count, cores, int(os.environ.get("ORACLE_POOL_MAX", "32"))))


def oracle_forwards(spec, indices, workers: int | None = None):
    """{b: (oracle output residues, scale, max |decrypt - float64|)} for every b in indices, computed by
    a spawn pool (the decryption error over the valid output slots of b, or of every item of b)."""
    indices = [int(b) for b in indices]
    workers = workers or workers_for(len(indices))
    ctx = mp.get_context("spawn")
    with cf.ProcessPoolExecutor(max_workers=workers, mp_context=ctx, initializer=_init, initargs=(spec,)) as ex:
        return {b: (d, s, e) for b, d, s, e in ex.map(_run, indices)}


def batch_messages(spec, count):
    s = setup(spec, keys=False)
    return s, np.stack([s["message"](b) for b in range(count)])

"""profiles/traffic.json from the committed ncu --set full exports (profiles/r02/final/prof_*_raw.csv): measured DRAM
bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, units from the CSV's unit row) beside the
algorithmic bytes of the same launch (DESIGN.md section 6 definitions).  bench.py reads the result."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = os.path.join(ROOT, "profiles", "r02", "final")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
N8 = 16384 * 8
B = 256


def rows(tag):
    r = list(csv.reader(open(os.path.join(D, f"prof_{tag}_raw.csv"))))
    h, u = r[0], r[1]
    out = []
    for vals in r[2:]:
        d = dict(zip(h, vals))
        un = dict(zip(h, u))
        byts = sum(float(d[k]) * UNIT[un[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        t = float(d["gpu__time_duration.sum"]) * {"us": 1e-3, "ms": 1.0, "ns": 1e-6, "s": 1e3}[un["gpu__time_duration.sum"]]
        out.append((d["Kernel Name"].split("(")[0].replace("void ", ""), d["Grid Size"], byts, t))
    return out


def entry(tag, alg, launch, idx=0):
    name, grid, byts, ms = rows(tag)[idx]
    return {"dram_bytes_per_launch": int(byts), "alg_bytes_per_launch": int(alg), "ratio": round(byts / alg, 3),
            "launch": f"{name} grid {grid}: {launch}", "duration_ms_under_ncu": round(ms, 4),
            "source": f"profiles/r02/final/prof_{tag}_raw.csv (ncu --set full, one launch)"}


nl, K, nd, G = 8, 2, 5, 8
ne = nl + K
out = {
    # baby-step IP, dense1 group: ModUp words of the non-own (digit, row) pairs + the input limbs (own rows and the
    # c0 addend) + keys read, G rotated Q_l P ciphertexts written
    "k_ks_ip_mma": entry("ipmma3", (B * (nd * ne - nl) + 2 * B * nl + G * nd * 2 * ne + G * B * 2 * ne) * N8,
                         "hybrid KS (dnum 5, K = 2), B = 256, nl = 8 (10 QP rows), G = 8 (dense1 baby-step group)"),
    # ModUp of the 2-prime digits of a giant step (all_e): 3 digits x 2 words read, 3 x 10 rows written
    "k_ks_modup": entry("modup2", (B * 3 * 2 + B * 3 * ne) * N8,
                        "giant-step ModUp of the three 2-prime digits to all 10 rows, B = 256"),
    # Eq. 1 sums of dense1: baby steps + input (t1 x B x 2) and plaintexts (t1 x t2) read, t2 x B x 2 written, per row
    "k_bsgs_mac_mma": entry("macmma", (64 * B * 2 + 64 * 8 + 8 * B * 2) * ne * N8,
                            "dense1 chunk, B = 256, t1 = 64, t2 = 8, all 10 QP rows (one launch)"),
    # giant-step IP, 4 steps in one accumulator pass: per step ModUp words (nd x ne), key and the sigma_g(w.c0)
    # addend (ne); the accumulator read + written once (2 x 2 x ne)
    "k_ks_ip_giant": entry("ipgiant", (4 * (B * nd * ne + nd * 2 * ne + B * ne) + 2 * 2 * B * ne) * N8,
                           "B = 256, nl = 8 (10 QP rows), giant steps 1-4 of dense1 in one pass"),
    # digits of a giant step: the 8 data limbs + 2 remainder words read per ciphertext, 8 digit words written
    "k_ks_digits": entry("digits", (B * nl + B * K + B * nl) * N8,
                         "giant-step digits (both sizes in one launch, QP input: fused ModDown), B = 256"),
    "k_ntt_batch_fwd": entry("nttbatch", 2 * 1024 * 8 * N8, "cfg2 forward, CTA pairs (cluster), TMA row stores", 0),
    "k_ntt_batch_inv": entry("nttbatch", 2 * 1024 * 8 * N8, "cfg2 inverse, CTA pairs (cluster)", 1),
}
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps({k: (v["ratio"], v["duration_ms_under_ncu"]) for k, v in out.items()}, indent=1))

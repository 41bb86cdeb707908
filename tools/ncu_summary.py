"""Summarise ncu CSV exports (raw page) and launch lists into profiles/ (committed evidence).

  python tools/ncu_summary.py raw  <kernel>_raw.csv [more...]      -> key metrics per kernel (json)
  python tools/ncu_summary.py launches launches.csv                  -> per-kernel time shares (json)
"""
import csv
import collections
import json
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum", "smsp__inst_executed.sum",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
]


def raw(paths):
    out = {}
    for p in paths:
        rows = list(csv.reader(open(p)))
        h, units = rows[0], rows[1]
        for vals in rows[2:]:
            d = dict(zip(h, vals))
            name = d.get("Kernel Name", p).split("(")[0]
            rec = {k: d[k] for k in KEYS if k in d}
            stalls = []
            for k, v in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            rec["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(stalls, reverse=True)[:6]}
            out[name] = rec
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        try:
            v = float(r[mi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    return {"total_ms": round(T / 1e6, 3),
            "kernels": {k: {"launches": cnt[k], "ms": round(v / 1e6, 3), "share": round(v / T, 4),
                            "avg_us": round(v / cnt[k] / 1e3, 1)} for k, v in sorted(tot.items(), key=lambda x: -x[1])}}


if __name__ == "__main__":
    mode, args = sys.argv[1], sys.argv[2:]
    print(json.dumps(raw(args) if mode == "raw" else launches(args[0]), indent=1))

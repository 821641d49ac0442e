"""Summarise an ncu report (read here, no GPU): per kernel launch, the metrics the
roofline needs.  Usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("sm_ghz", "sm__cycles_elapsed.avg.per_second"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_mem_pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("l1tex_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "Ghz": 1.0, "Mhz": 1e-3}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, m in KEYS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    v = r[i]
                d[k] = round(v, 3) if isinstance(v, float) else v
        res.append(d)
    return res


def stalls(path, top=8):
    """Share of warp-stall samples by reason and the hottest SASS lines (needs --import-source)."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (KeyError, ValueError):
            return 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1.0
    reasons = {h[6:]: round(100 * sum(f(r, h) for r in data) / tot, 1) for h in hdr
               if h.startswith("stall_") and "Not Issued" not in h}
    hot = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]
    return {"stall_pct_by_reason": {k: v for k, v in sorted(reasons.items(), key=lambda kv: -kv[1]) if v > 0.5},
            "hottest_sass": [(round(100 * f(r, "Warp Stall Sampling (All Samples)") / tot, 1), r[ix["Source"]].strip())
                             for r in hot]}


if __name__ == "__main__":
    res = load(sys.argv[1])
    if "--stalls" in sys.argv:
        st = stalls(sys.argv[1])
        for d in res:
            d["stalls"] = st
    for d in res:
        print(json.dumps(d))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)

"""Per-kernel-family time share and achieved DRAM bandwidth from an ncu CSV launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (cold, serialised).
Usage: python tools/ncu_launch_bw.py launches.csv [--top 25] [--json out.json]"""
import collections
import csv
import json
import sys

TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
BYTES = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}


def family(name):
    if "gemm_kernel" in name:
        i = name.index("gemm_kernel")
        return name[i:name.index(">", i) + 1]
    return name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").strip()


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(lambda: {"launches": set(), "us": 0.0, "MB": 0.0})
    for r in rows[hi + 1:]:
        try:
            name, met, unit = r[ix["Kernel Name"]], r[ix["Metric Name"]], r[ix["Metric Unit"]]
            val = float(r[ix["Metric Value"]].replace(",", ""))
        except (IndexError, ValueError, KeyError):
            continue
        f = per[family(name)]
        f["launches"].add(r[ix["ID"]])
        if met == "gpu__time_duration.sum":
            f["us"] += val * TIME.get(unit, 1e-3)
        elif met in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            f["MB"] += val * BYTES.get(unit, 1e-6)
    tot = sum(f["us"] for f in per.values()) or 1.0
    out = []
    for k, f in sorted(per.items(), key=lambda kv: -kv[1]["us"]):
        out.append({"kernel": k, "launches": len(f["launches"]), "us": round(f["us"], 1),
                    "share": round(f["us"] / tot, 4), "MB": round(f["MB"], 1),
                    "TB_per_s": round(f["MB"] / f["us"], 3) if f["us"] else None})   # MB/us = TB/s
    return out, tot


if __name__ == "__main__":
    res, tot = load(sys.argv[1])
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    for d in res[:top]:
        print(f"{100 * d['share']:5.1f}%  n={d['launches']:4d}  {d['us']:9.1f} us  {d['MB']:9.1f} MB  "
              f"{d['TB_per_s']:6.2f} TB/s  {d['kernel']}")
    print(f"total {tot:.1f} us")
    if "--json" in sys.argv:
        json.dump({"total_us": tot, "kernels": res}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)

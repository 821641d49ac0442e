"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list by kernel family.
Usage: python tools/launches_summary.py launches.csv out.json "<source description>" """
import collections
import csv
import json
import sys

FAMILIES = ["gemm_kernel<256, 0, 0, 0>", "gemm_kernel<256, 0, 1, 0>", "gemm_kernel<256, 1, 1, 0>",
            "gemm_kernel<128, 0, 1, 1>", "gemm_kernel<64", "gemm_kernel<128", "sgd_update", "bias_grad_fused", "bias_grad_partial",
            "bias_grad_final", "softmax", "loss_mean", "fill_synthetic", "f32_to_bf16", "nccl"]
LABEL = {"gemm_kernel<256, 0, 0, 0>": "gemm fwd (BN=256)", "gemm_kernel<256, 0, 1, 0>": "gemm dgrad (BN=256)",
         "gemm_kernel<256, 1, 1, 0>": "gemm wgrad (BN=256)", "gemm_kernel<128, 0, 1, 1>": "gemm dgrad blend-on-load"}
UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def family(name):
    """gemm_kernel<BN, A_MN, B_MN, BLEND, SGD, CG, CONV> -> readable label; other kernels by prefix."""
    import re
    m = re.search(r"gemm_kernel<\s*(\d+),\s*(\d),\s*(\d),\s*(\d),\s*(\d),\s*(\d),\s*(\d)>", name.replace("(int)", ""))
    if m:
        bn, amn, bmn, blend, sgd, cg, conv = (int(x) for x in m.groups())
        kind = {(0, 0): "fwd", (0, 1): "dgrad", (1, 1): "wgrad"}[(amn, bmn)]
        if conv:
            kind = "conv " + kind
        if blend:
            kind += " blend-on-load"
        if sgd:
            kind += "+update"
        return f"gemm {kind} (BN={bn}, {'CTA pair' if cg == 2 else '1 CTA'})"
    return next((f for f in FAMILIES if f in name), name[:50])


def main(path, out, src):
    rows = list(csv.reader(open(path)))
    hi = next((i for i, r in enumerate(rows) if "Kernel Name" in r), None)
    if hi is None:   # ncu captured nothing (the profiled program failed): say so instead of a traceback
        raise SystemExit(f"{path}: no kernel rows (did the profiled command fail? see its log)")
    hdr = rows[hi]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = family(r[ki])
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    res = {k: {"launches": v[0], "us_total": round(v[1], 1), "us_per_launch": round(v[1] / v[0], 2),
               "share": round(v[1] / tot, 4)} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    json.dump({"source": src, "note": "ncu per-launch times are cold-cache and serialised: compare shares",
               "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")

"""Per-kernel share of GPU time from an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_list.py gpurun_out/tNN/launches.csv "<command description>" > profiles/...json
"""
import csv
import json
import sys


def main():
    path, source = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(path)) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[head]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = {}
    for r in rows[head + 1:]:
        if len(r) <= max(ki, mi, vi) or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        if "xpgb" not in name:
            continue
        us = float(r[vi].replace(",", "")) * (scale.get(r[ui], 1.0) if ui is not None else 1e-3)
        a = agg.setdefault(name, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += us
    tot = sum(a["total_us"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["share"] = a["total_us"] / tot
    out = {"source": source, "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Summarise an ncu report into the numbers the roofline needs (per launch).

    python tools/ncu_summary.py gpurun_out/r1/gate_up.ncu-rep [--algo-bytes N]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "Kbyte/block": 1e3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:80] if "Kernel Name" in hdr else None}
        for i, h in enumerate(hdr):
            if h in KEYS:
                v = vals[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
                rec[KEYS[h]] = v
        if "dram_read" in rec and "dram_write" in rec:
            rec["traffic_bytes"] = rec["dram_read"] + rec["dram_write"]
            rec["dram_gbps"] = rec["traffic_bytes"] / rec["duration"] / 1e9
        out.append(rec)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    algo = None
    if "--algo-bytes" in sys.argv:
        algo = float(sys.argv[sys.argv.index("--algo-bytes") + 1])
    for r in res:
        if algo:
            r["algorithmic_bytes"] = algo
            r["traffic_over_algorithmic"] = r["traffic_bytes"] / algo
        print(json.dumps(r))

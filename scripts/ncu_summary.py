"""Summarise an ncu report (``ncu -i R.ncu-rep --page raw --csv > R.csv``) as
one JSON object per profiled launch with the metrics the roofline needs.

    python scripts/ncu_summary.py R.csv > profiles/<name>.json
"""
import csv
import json
import sys

WANT = {
    "duration_us": ("gpu__time_duration.sum", None),  # scaled to us from the unit row
    "dram_read_B": ("dram__bytes_read.sum", None),
    "dram_write_B": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", None),
    "fma_pipe_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "smem_per_block_B": ("launch__shared_mem_per_block", None),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3, "byte/block": 1,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    names, units = rows[head], rows[head + 1]
    col = {n: i for i, n in enumerate(names)}
    out = []
    for r in rows[head + 2:]:
        if len(r) != len(names):
            continue
        rec = {"kernel": r[col["Kernel Name"]][:80]}
        for key, (metric, _) in WANT.items():
            if metric not in col:
                continue
            v = r[col[metric]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                rec[key] = v
                continue
            u = units[col[metric]]
            if key == "duration_us":
                x *= SCALE[u]
            elif key.endswith("_B"):
                x *= SCALE[u]
            rec[key] = x
        out.append(rec)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])

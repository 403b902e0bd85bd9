"""Summarise ncu captures into profiles/ (markdown + json), run here (no GPU)."""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
        "launch__shared_mem_per_block_dynamic"]


def full_report(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append({"kernel": d.get("Kernel Name", "").split("(")[0],
                    **{k: (d[k], units[hdr.index(k)]) for k in KEYS if k in d}})
    return res


def launch_list(path: str) -> list[tuple]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "us": 1.0, "ns": 1e-3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [(k, n, us, us / tot) for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    mode, src, dst = sys.argv[1], sys.argv[2], sys.argv[3]
    if mode == "full":
        data = full_report(src)
        Path(dst).write_text(json.dumps(data, indent=1) + "\n")
        for d in data:
            print(d["kernel"])
            for k in KEYS:
                if k in d:
                    print(f"  {k} = {d[k][0]} {d[k][1]}")
    else:
        rows = launch_list(src)
        lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
        lines += [f"| {k} | {n} | {us:.1f} | {100*s:.1f}% |" for k, n, us, s in rows]
        Path(dst).write_text("\n".join(lines) + "\n")
        print("\n".join(lines))

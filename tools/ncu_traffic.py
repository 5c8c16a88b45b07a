"""Summarise an `ncu --set full` capture into profiles/<round>/ncu_traffic.json:
per kernel, launches, average duration, DRAM bytes (read + write) per launch
and tensor-pipe utilisation. bench.py reads `dram_bytes_per_launch` for its
roofline `traffic` field.

usage: python tools/ncu_traffic.py REP.ncu-rep OUT.json "source description"
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "rd",
    "dram__bytes_write.sum": "wr",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tc",
}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9, "%": 1.0, "": 1.0}

KEYS = {"gemm2_kernel": "gemm::gemm2_kernel", "gemm_kernel<256>": "gemm::gemm_kernel<256>",
        "gemm_kernel<128>": "gemm::gemm_kernel<128>", "attn_fwd_kernel": "attn::attn_fwd_kernel",
        "attn_bwd_kernel": "attn::attn_bwd_kernel", "fetch_tma_kernel": "fetch_tma_kernel",
        "push_red_kernel": "push_red_kernel", "adam_kernel": "adam_kernel"}


def short(name):
    for k, v in KEYS.items():
        if k in name:
            return v
    return None


def main(rep, out, source):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if not l.startswith("==")))))
    head, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(head)}
    for h, i in list(col.items()):  # section-prefixed names ("TPC.TriageCompute.<metric>")
        col.setdefault(h.split(".", 2)[-1] if h.count(".") >= 2 and h.split(".")[0].isupper() else h, i)
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        k = short(r[col["Kernel Name"]])
        if k is None:
            continue
        for m, tag in METRICS.items():
            if m in col and r[col[m]] not in ("", "n/a", "no data"):
                acc[k][tag].append(float(r[col[m]].replace(",", "")) * SCALE.get(units[col[m]], 1.0))
    res = {}
    for k, d in sorted(acc.items()):
        n = len(d["us"])
        res[k] = {"launches": n, "avg_us": round(sum(d["us"]) / n, 2),
                  "dram_bytes_per_launch": int(round((sum(d["rd"]) + sum(d["wr"])) / n)),
                  "tensor_pipe_pct_avg": round(sum(d["tc"]) / max(len(d["tc"]), 1), 1)}
    with open(out, "w") as f:
        json.dump({"source": source, "kernels": res}, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])

"""Summarise an `ncu --set full` capture of tools/ncu_step_kernels.py into
profiles/<round>/ncu_traffic.json: per kernel, launches, average duration,
DRAM bytes (read + write) per launch and tensor activity; per GEMM launch its
(M, N, K) (from gpurun_out/ncu_gemm_launches.json, written by the capture
tool in launch order), algorithmic TFLOP/s = 2MNK / duration, and the
counter-based TFLOP/s = sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum /
duration — the two must agree (the ops counter counts what the tensor pipe
executed). bench.py reads `dram_bytes_per_launch` for its roofline `traffic`.

usage: python tools/ncu_traffic.py REP.ncu-rep OUT.json "source description" [gemm_launches.json]
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
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum": "ops",
    "sm__inst_executed_pipe_tc.sum": "tcinst",
}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9, "%": 1.0, "": 1.0}

KEYS = {"gemm2_kernel": "gemm::gemm2_kernel", "gemm_kernel<256>": "gemm::gemm_kernel<256>",
        "gemm_kernel<128>": "gemm::gemm_kernel<128>", "attn_fwd_kernel": "attn::attn_fwd_kernel",
        "attn_bwd_kernel": "attn::attn_bwd_kernel", "fetch_tma_kernel": "fetch_tma_kernel",
        "push_red_kernel": "push_red_kernel", "push_bulk_kernel": "push_bulk_kernel", "adam_kernel": "adam_kernel",
        "slot_reduce_kernel": "slot_reduce_kernel", "fixed_finalize_kernel": "fixed_finalize_kernel"}


def short(name):
    for k, v in KEYS.items():
        if k in name:
            return v
    return None


def main(rep, out, source, launches=None):
    """rep: an .ncu-rep, or the CSV of `ncu -i REP --page raw --csv` exported on the GPU box."""
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if not l.startswith("==")))))
    head, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(head)}
    for h, i in list(col.items()):  # section-prefixed names ("TPC.TriageCompute.<metric>")
        col.setdefault(h.split(".", 2)[-1] if h.count(".") >= 2 and h.split(".")[0].isupper() else h, i)
    acc = defaultdict(lambda: defaultdict(list))
    gemm_rows = []
    for r in rows[2:]:
        k = short(r[col["Kernel Name"]])
        if k is None:
            continue
        vals = {}
        for m, tag in METRICS.items():
            if m in col and r[col[m]] not in ("", "n/a", "no data"):
                vals[tag] = float(r[col[m]].replace(",", "")) * SCALE.get(units[col[m]], 1.0)
                acc[k][tag].append(vals[tag])
        if k.startswith("gemm::"):
            gemm_rows.append(vals)
    res = {}
    for k, d in sorted(acc.items()):
        n = len(d["us"])
        res[k] = {"launches": n, "avg_us": round(sum(d["us"]) / n, 2),
                  "dram_bytes_per_launch": int(round((sum(d["rd"]) + sum(d["wr"])) / n)),
                  "tensor_pipe_pct_avg": round(sum(d["tc"]) / max(len(d["tc"]), 1), 1) if d["tc"] else None}
        if d["ops"] and sum(d["ops"]) > 0:
            res[k]["counter_tflops_avg"] = round(sum(d["ops"]) / (sum(d["us"]) * 1e6), 1)
    per_launch = []
    if launches:
        shapes = json.load(open(launches))
        for i, (v, s) in enumerate(zip(gemm_rows, shapes)):
            alg = s["flops"] / (v["us"] * 1e6)
            row = {"i": i, "kind": s["kind"], "M": s["M"], "N": s["N"], "K": s["K"], "us": round(v["us"], 1),
                   "alg_tflops": round(alg, 1), "dram_MB": round((v.get("rd", 0) + v.get("wr", 0)) / 1e6, 1)}
            if v.get("ops"):
                row["counter_tflops"] = round(v["ops"] / (v["us"] * 1e6), 1)
                row["counter_over_alg"] = round(row["counter_tflops"] / alg, 3)
            per_launch.append(row)
    with open(out, "w") as f:
        json.dump({"source": source, "kernels": res, "gemm_launches": per_launch}, f, indent=1)
    print(json.dumps(res, indent=1))
    for row in per_launch:
        print(json.dumps(row))


if __name__ == "__main__":
    main(*sys.argv[1:5])

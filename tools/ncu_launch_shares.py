"""Per-kernel share of device time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv <cmd>`):
launches, total and average duration, share of the summed device time. ncu
serialises and cold-starts every launch, so the absolute times are not the
bench's; the SHARES are what agree with the event-timed step.

usage: python tools/ncu_launch_shares.py L.csv [OUT.txt]
"""
import csv
import io
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def main(path, out=None):
    txt = [l for l in open(path).read().splitlines() if not l.startswith("==")]
    rows = list(csv.reader(io.StringIO("\n".join(txt))))
    head = rows[0]
    ci = {k: i for i, k in enumerate(head)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) < len(head) or r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ci["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        ms = float(r[ci["Metric Value"]].replace(",", "")) * SCALE.get(r[ci["Metric Unit"]], 1.0)
        agg[short][0] += 1
        agg[short][1] += ms
    total = sum(v[1] for v in agg.values())
    lines = [f"total device time {total:.2f} ms over {sum(v[0] for v in agg.values())} launches (ncu, serialised)"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{100 * ms / total:6.2f}%  {ms:9.3f} ms  n={n:5d}  avg {1e3 * ms / n:9.1f} us  {k}")
    text = "\n".join(lines)
    print(text)
    if out:
        with open(out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:3])

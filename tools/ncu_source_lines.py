"""Per-source-line warp-stall attribution of one kernel from an ncu capture's
SASS source page (`ncu -i REP --page source --csv --print-source sass`),
mapped to CUDA lines with `nvdisasm -g` of the same build's cubin (ncu's own
CUDA view of a -lineinfo build carries no metrics here).

usage: python tools/ncu_source_lines.py SOURCE_SASS.csv[.gz] KERNEL_CUBIN MANGLED_NAME SRC.cu [top]
"""
import collections
import csv
import gzip
import io
import re
import subprocess
import sys


def main(src_csv, cubin, fn, cu, top=30):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
    start = [k for k, l in enumerate(dis) if l.startswith("//--------------------- .text." + fn)][0]
    cur, off2line = None, {}
    for l in dis[start + 1:]:
        if l.startswith("//--------------------- .text"):
            break
        m = re.search(r'//## File ".*?", line (\d+)', l)
        if m:
            cur = int(m.group(1))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    f = gzip.open(src_csv, "rt") if src_csv.endswith(".gz") else open(src_csv)
    rows = list(csv.reader(io.StringIO(f.read())))
    head = rows[1]
    ci = {h: k for k, h in enumerate(head)}
    stalls = [h for h in head if h.startswith("stall_") and "Not Issued" not in h]
    base = int(rows[2][0], 16)
    byline, bystall = collections.Counter(), collections.defaultdict(collections.Counter)
    for r in rows[2:]:
        ln = off2line.get(int(r[0], 16) - base)
        v = r[ci["Warp Stall Sampling (All Samples)"]]
        byline[ln] += int(v) if v.isdigit() else 0
        for s in stalls:
            if r[ci[s]].isdigit():
                bystall[ln][s[6:]] += int(r[ci[s]])
    src = open(cu).read().split("\n")
    tot = sum(byline.values())
    for ln, n in byline.most_common(int(top)):
        txt = src[ln - 1].strip()[:72] if ln else "?"
        print(f"{n:8d} {100 * n / tot:5.1f}%  L{ln}: {txt:72s} {bystall[ln].most_common(2)}")


if __name__ == "__main__":
    main(*sys.argv[1:6])

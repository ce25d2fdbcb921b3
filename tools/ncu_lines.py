"""Summarise an `ncu --page source --csv --print-source cuda,sass` export:
per CUDA source line, executed warp instructions and warp-stall samples.

    python tools/ncu_lines.py c3_source.csv.gz [top]
"""
import csv
import gzip
import io
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    op = gzip.open if path.endswith(".gz") else open
    text = op(path, "rt").read()
    rows = []
    fname = None
    stats = {}
    for r in csv.reader(io.StringIO(text)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            if r[0] == "Line No":
                hdr = r
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        if r[2] != "-":  # sass rows carry an address; the cuda rows aggregate
            continue
        key = (fname, line)
        samp = int(r[4] or 0)
        inst = int(r[7] or 0)
        s = stats.setdefault(key, [0, 0, r[1][:90]])
        s[0] += samp
        s[1] += inst
    tot_s = sum(v[0] for v in stats.values()) or 1
    tot_i = sum(v[1] for v in stats.values()) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / tot_s:5.1f}% smp {100 * v[1] / tot_i:5.1f}% ins  {k[0]}:{k[1]:<5} {v[2]}")


if __name__ == "__main__":
    main()

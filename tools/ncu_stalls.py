"""Stall-reason breakdown per CUDA source line from an
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` export.

    python tools/ncu_stalls.py src.csv [file:line ...]   (no lines: totals)
"""
import collections
import csv
import io
import sys


def main():
    rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read())))
    want = set(sys.argv[2:])
    hdr = None
    tot = collections.Counter()
    per = collections.defaultdict(collections.Counter)
    fname = None
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Address"] != "-":  # sass rows repeat the line totals: use source rows only
            continue
        key = f"{fname}:{d['Line No']}" if fname else d["Line No"]
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    x = float(v)
                except ValueError:
                    continue
                tot[k] += x
                per[key][k] += x
    print("total:", {k: int(v) for k, v in tot.most_common(12)})
    for w in want:
        print(w, {k: int(v) for k, v in per[w].most_common(8)})


if __name__ == "__main__":
    main()

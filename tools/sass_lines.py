"""Per-source-line SASS instruction counts of one kernel in a cubin/object
(nvdisasm -g line info), for checking what the compiler made of a loop.

    python tools/sass_lines.py build/fit_big.o <kernel-substring> [lo hi]
"""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main():
    obj, key = sys.argv[1], sys.argv[2]
    lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=d, check=True,
                       capture_output=True)
        cub = next(Path(d).glob("*.cubin"))
        out = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout
    func = cur = None
    cnt = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.search(r'\.text\.(\S+):', line)
        if m:
            func = m.group(1)
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1), int(m.group(2)))
        m = re.search(r'/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', line)
        if m and func and key in func and cur:
            cnt[cur] += 1
            ops[cur][m.group(1).split('.')[0]] += 1
    print("total", sum(cnt.values()))
    for k in sorted(cnt, key=lambda k: (k[0], k[1])):
        if lo <= k[1] <= hi:
            print(f"{k[0]}:{k[1]:<5} {cnt[k]:6d}  {dict(ops[k].most_common(5))}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Warp-stall samples of one kernel per CUDA source line.

ncu's source page (--print-source sass) gives samples per SASS address; the
line table comes from nvdisasm -g on the built object (compiled -lineinfo).

  python tools/ncu_sass_lines.py <report.ncu-rep> <object.o> <kernel-substring> [top]
"""
import csv
import io
import re
import subprocess
import sys
import tempfile
import os


def sass_samples(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    res = []
    for r in rows[2:]:
        if len(r) <= iss:
            continue
        res.append((int(r[ia], 16), r[isrc].strip(), int(r[iss] or 0)))
    base = res[0][0]
    return [(a - base, s, n) for a, s, n in res]


def line_table(obj, kern):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout
    table, cur, infn = {}, None, False
    for line in dis.splitlines():
        if re.match(r"\s*\.text\.", line) or line.startswith(".section"):
            infn = kern in line
        m = re.search(r'//## File "(.*)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        a = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if a and infn:
            table[int(a.group(1), 16)] = cur
    return table


def main():
    rep, obj, kern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    samples = sass_samples(rep)
    table = line_table(obj, kern)
    per = {}
    total = 0
    for a, s, n in samples:
        key = table.get(a, ("?", 0))
        e = per.setdefault(key, [0, {}])
        e[0] += n
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        e[1][op] = e[1].get(op, 0) + n
        total += n
    print(f"total samples {total}")
    for key, (n, ops) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        tops = ", ".join(f"{o} {c}" for o, c in sorted(ops.items(), key=lambda kv: -kv[1])[:3])
        print(f"{n:6d} {100.0 * n / total:5.1f}%  {key[0]}:{key[1]}  [{tops}]")


if __name__ == "__main__":
    main()

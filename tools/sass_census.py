#!/usr/bin/env python3
"""Per-kernel SASS instruction census of the built library: the mnemonics that
prove the Blackwell-native path (UTCHMMA / UTCQMMA tensor-core MMAs, UTMALDG /
UTMASTG / UTMAREDG TMA, LDTM / STTM TMEM, UTCBAR commits) next to the legacy
HMMA and the MUFU / FFMA2 softmax work.

  python tools/sass_census.py [lib.so] > profiles/r02_sass_census.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2602_07309_b200", "lib",
                                                          "libsemrank_b200.so")
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF", "UBLKCP", "LDTM",
        "STTM", "HMMA", "MUFU.EX2", "FFMA2", "FMUL2", "FADD2", "FMNMX3", "SYNCS"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
func = None
counts = collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        func = m.group(1)
        counts[func] = collections.Counter()
        continue
    if func is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            counts[func][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(.*", "", d)
    d = d.replace("srk::", "").replace("(anonymous namespace)::", "")
    return d[:90]


print("# SASS instruction census per kernel (static counts), "
      f"`{os.path.relpath(LIB, ROOT)}`\n")
print("`cuobjdump -sass` of the built library, summarised by `tools/sass_census.py`. Static "
      "instruction counts (not executed counts); kernels with none of the listed mnemonics "
      "are omitted.\n")
print("| kernel | " + " | ".join(KEYS) + " |")
print("|---|" + "---|" * len(KEYS))
for f, c in counts.items():
    if not any(c.values()):
        continue
    print(f"| `{short(f)}` | " + " | ".join(str(c[k]) if c[k] else "" for k in KEYS) + " |")

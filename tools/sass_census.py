#!/usr/bin/env python
"""SASS census of libs3.so: per kernel, how many instructions of the
mnemonics that prove the Blackwell paths (tcgen05 MMA / TMEM loads and
stores, TMA tensor loads and stores, bulk copies, mbarrier sync) and the
CUDA-core math.  Runs on the build host (cuobjdump, no GPU needed).

    python tools/sass_census.py [path/to/libs3.so]
"""
from __future__ import annotations

import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF", "UBLKCP", "SYNCS",
        "HMMA", "FFMA", "MUFU.EX2", "SHFL", "LDS", "LDG", "STG", "REDG", "ATOMG", "ELECT", "FENCE"]


def census(lib):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True,
                          check=True).stdout
    per = collections.OrderedDict()
    arch = None
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*arch = (sm_\w+)", line)
        if m:
            arch = m.group(1)
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    per[cur][k] += 1
    return arch, per


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
        return out[:len(names)]
    except Exception:
        return names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2306_06000_b200", "lib", "libs3.so")
    arch, per = census(lib)
    print(f"# SASS census of {os.path.relpath(lib, ROOT)} ({arch}); counts of static instructions per kernel")
    names = demangle(list(per))
    for (raw, cnt), name in zip(per.items(), names):
        short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", "")).replace("s3::", "")
        got = ", ".join(f"{k} {cnt[k]}" for k in KEYS if cnt[k])
        print(f"{short:40s} {got}")


if __name__ == "__main__":
    main()

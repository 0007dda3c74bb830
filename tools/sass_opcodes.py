#!/usr/bin/env python
"""Per-kernel SASS opcode counts of the built library (cuobjdump -sass), the
evidence that the hot path is tcgen05 / TMA / mma.sync code.
usage: python tools/sass_opcodes.py [lib] > profiles/rN/sass_opcodes.txt"""
import re
import subprocess
import sys
from collections import Counter

OPS = ["UTMALDG", "UBLKCP", "UTMASTG", "HMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "LDSM", "LDS", "STS",
       "PRMT", "LOP3", "SHF", "HMUL2", "SYNCS", "FENCE", "MEMBAR"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2407_10960_b200/libflute_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    demangled = subprocess.run(["c++filt"], input=sass, capture_output=True, text=True).stdout
    print(f"# SASS opcode counts per kernel (cuobjdump -sass {lib})")
    print("# UTMALDG = TMA tensor load, UBLKCP = bulk copy, HMMA = mma.sync, UTCHMMA = tcgen05.mma, "
          "LDTM/STTM = tcgen05.ld/st, UTCBAR = tcgen05.commit")
    print("kernel | total | " + " | ".join(OPS))
    name, cnt, tot = None, Counter(), 0
    def flush():
        if name:
            print(f"{name[:90]} | {tot} | " + " | ".join(str(cnt[o]) for o in OPS))
    for line in demangled.splitlines():
        m = re.match(r"\s+Function : (.*)", line)
        if m:
            flush()
            name, cnt, tot = m.group(1).replace("flute_dev::", ""), Counter(), 0
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and name:
            tot += 1
            cnt[m.group(1)] += 1
    flush()


if __name__ == "__main__":
    main()

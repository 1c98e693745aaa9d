"""Per-kernel SASS instruction counts of libsgrpo_b200.so (cuobjdump -sass): the evidence of which
kernels run on the Blackwell-native paths (UTC*MMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG /
UBLKCP = TMA / bulk copies) vs the legacy tensor path (HMMA = mma.sync).

    python scripts/sass_counts.py > profiles/r02_sass_counts.txt
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2509_21792_b200",
                   "libsgrpo_b200.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "HMMA", "LDSM", "MOVM",
       "DFMA", "DADD", "DMUL"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    fn = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        if fn is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[A-Z0-9_.]+)?\b", line)
        if m:
            counts[fn][m.group(1)] += 1
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    print("# cuobjdump -sass paper_2509_21792_b200/libsgrpo_b200.so: instruction counts per kernel")
    print("# columns: " + " ".join(OPS) + " | total | kernel")
    for (fn, c), name in zip(counts.items(), names):
        short = name.replace("(anonymous namespace)::", "")
        short = re.sub(r"\(.*", "", short)
        tot = sum(c.values())
        print(" ".join(f"{c[o]:6d}" for o in OPS) + f" | {tot:6d} | {short}")


if __name__ == "__main__":
    sys.exit(main())

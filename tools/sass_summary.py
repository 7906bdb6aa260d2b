"""Per-kernel SASS opcode counts of the in-tree libnpm.so (the evidence that
the kernels are Blackwell-native: UTC*MMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st,
UBLKCP/UTMALDG = TMA, REDG = vector reductions).  usage: python tools/sass_summary.py [lib] > out.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "REDG", "LDG", "STG", "LDS", "STS", "BAR",
        "SYNCS", "MUFU", "HMMA", "STL", "LDL"]


def main(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kern, counts = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts.setdefault(kern, collections.Counter())
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and kern:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    counts[kern][k] += 1
    demangle = lambda s: subprocess.run(["c++filt", s], capture_output=True, text=True).stdout.strip()
    total = collections.Counter()
    print("# SASS opcode counts per kernel of %s (cuobjdump -sass)" % os.path.relpath(lib, ROOT))
    print("# columns: " + " ".join(KEYS))
    for kern, c in counts.items():
        total.update(c)
        name = demangle(kern)
        name = re.sub(r"npm::detail::Net<\(int\)(\d+), \(int\)(\d+), \(int\)(\d+), \(int\)(\d+)>", r"Net<\1,\2,\3,\4>", name)
        print("%-100s %s" % (name[:100], " ".join("%s=%d" % (k, c[k]) for k in KEYS if c[k])))
    print("TOTAL " + " ".join("%s=%d" % (k, total[k]) for k in KEYS))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2504_04315_b200", "libnpm.so"))

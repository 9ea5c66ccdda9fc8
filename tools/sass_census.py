"""Per-kernel SASS census of libhmx.so: tensor-core (DMMA), bulk-copy / TMA (UBLKCP, UTMALDG),
mbarrier (SYNCS), Ampere-style async copies (LDGSTS), FP64 (DFMA / DADD / DMUL) instruction counts.

    python tools/sass_census.py [path/to/libhmx.so] > profiles/rNN_sass_census.txt
"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1706_09384_b200/libhmx.so"
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["DMMA", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "LDGSTS", "DFMA", "DADD", "DMUL", "LDS", "LDG", "STG"]
kern, counts, order = None, {}, []
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = dict.fromkeys(OPS, 0)
        order.append(kern)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+)", line)
    if kern and m:
        op = m.group(1)
        if op in counts[kern]:
            counts[kern][op] += 1


def short(name):
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    dem = re.sub(r"hmx::\(anonymous namespace\)::", "", dem)
    return dem.split("(")[0]


print("kernel".ljust(58) + "".join(o.rjust(8) for o in OPS))
for k in order:
    c = counts[k]
    if sum(c.values()) == 0:
        continue
    print(short(k)[:57].ljust(58) + "".join(str(c[o]).rjust(8) for o in OPS))

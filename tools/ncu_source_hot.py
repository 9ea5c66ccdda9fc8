"""Hot instructions of an `ncu --page source --csv` export: stall mix and the top sampled SASS lines.

    ncu -i prof.ncu-rep --page source --csv > src.csv; python tools/ncu_source_hot.py src.csv [ntop]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 45
hdr = rows[1]
data = []
for r in rows[2:]:  # the first kernel of the export only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
samp = [int(r[ix["# Samples"]]) for r in data]
inst = [int(r[ix["Instructions Executed"]]) for r in data]
tot = sum(samp)
print(rows[0][1][:100])
print("total samples", tot, "warp instructions", sum(inst))
agg = {s: sum(int(r[ix[s]]) for r in data) for s in stalls}
print("  " + "  ".join(f"{s[6:]} {100 * v / tot:.1f}%" for s, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
for i in sorted(sorted(range(len(data)), key=lambda i: -samp[i])[:ntop]):
    r = data[i]
    st = sorted(((int(r[ix[s]]), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{i:6d} {100 * samp[i] / tot:5.2f}%  {r[ix['Source']].strip()[:64]:64s} x{inst[i]:>10d}  {st}")

import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ai, si, ii, ti = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
items = []
for r in rows[2:]:
    try:
        items.append((float(r[ii] or 0), float(r[ti] or 0), r[ai], r[si]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in items) or 1
tots = sum(x[1] for x in items) or 1
print("instructions", tot, "samples", tots)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for x in sorted(items, key=lambda x: -x[1])[:n]:
    print("%5.1f%%i %5.1f%%s %s %s" % (100 * x[0] / tot, 100 * x[1] / tots, x[2], x[3][:90]))
# instruction mix by opcode
from collections import Counter
c = Counter()
for x in items:
    op = x[3].split()[0] if x[3] else "?"
    if op.startswith("@"):
        op = x[3].split()[1]
    c[op.split(".")[0]] += x[0]
print("opcode mix:", [(k, round(100 * v / tot, 1)) for k, v in c.most_common(18)])

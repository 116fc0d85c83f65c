"""Attribute ncu per-SASS-instruction counts / stall samples to source lines via nvdisasm -g."""
import csv, re, sys
from collections import defaultdict
sass_file, func, csv_file = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(sass_file).read().splitlines()
start = None
for i, l in enumerate(lines):
    if l.startswith(".text." + func + ":"):
        start = i
        break
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//---"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        if "inlined at" not in l:  # (file, line): the same line number in different headers must not merge
            cur = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_file)))
hdr = rows[1]
ai, ii, ti = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ai], 16), float(r[ii] or 0), float(r[ti] or 0)))
    except (ValueError, IndexError):
        pass
base = min(d[0] for d in data)
agg_i, agg_s = defaultdict(float), defaultdict(float)
for a, n, s in data:
    ln = off2line.get(a - base)
    agg_i[ln] += n
    agg_s[ln] += s
ti_, ts_ = sum(agg_i.values()), sum(agg_s.values())
src = open(sys.argv[4]).read().splitlines() if len(sys.argv) > 4 else None  # optional: the main source
for key in sorted(agg_i, key=lambda k: -agg_i[k])[:30]:
    f, ln = key if key else ("?", 0)
    txt = src[ln - 1].strip()[:80] if (src and ln and len(sys.argv) > 4 and sys.argv[4].endswith(f)) else ""
    print("%s:%-5s inst %5.1f%%  stall %5.1f%%  %s" % (f, ln, 100 * agg_i[key] / ti_, 100 * agg_s[key] / ts_, txt))

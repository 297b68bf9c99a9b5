"""Stall samples and instructions of an ncu SASS source CSV grouped by address regions.
usage: sass_regions.py <csv> name:start-end ...   (hex offsets, low 20 bits)"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r][0]
hdr = rows[hi]
si = hdr.index('Warp Stall Sampling (All Samples)'); ii = hdr.index('Instructions Executed')
scols = [(i, h) for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
regs = []
for a in sys.argv[2:]:
    n, rng = a.split(':'); lo, hi_ = rng.split('-'); regs.append((n, int(lo, 16), int(hi_, 16)))
seen = set(); agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= si or r[0] in seen: continue
    seen.add(r[0])
    try: a = int(r[0], 16) & 0xfffff; s = float(r[si] or 0); n = float(r[ii] or 0)
    except Exception: continue
    tot += s
    name = next((x[0] for x in regs if x[1] <= a <= x[2]), 'other')
    agg[name][0] += s; agg[name][1] += n
    for i, h in scols:
        try: agg[name][2][h[6:]] += float(r[i] or 0)
        except Exception: pass
for name, (s, n, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    top = ', '.join(f"{k} {v/s*100:.0f}%" for k, v in c.most_common(4)) if s else ''
    print(f"{name:10s} samples {s/tot*100:5.1f}%  inst {n:.3g}  [{top}]")

"""Top SASS instructions by stall samples from an ncu --page source CSV (tools/ncu_export.sh)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r][0]
hdr = rows[hi]
si = hdr.index('Warp Stall Sampling (All Samples)'); ii = hdr.index('Instructions Executed'); src = hdr.index('Source')
data = []
for r in rows[hi + 1:]:
    try: data.append((float(r[si] or 0), float(r[ii] or 0), r[0], r[src].strip()))
    except Exception: pass
ts = sum(d[0] for d in data) or 1; ti = sum(d[1] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print('samples', ts, 'warp-inst', ti)
op_st = collections.Counter(); op_in = collections.Counter()
for d in data:
    s = d[3]; op = (s.split()[1] if s.startswith('@') else s.split()[0]).split('.')[0] if s else '?'
    op_st[op] += d[0]; op_in[op] += d[1]
for op, v in op_st.most_common(12): print(f"  {op:10s} stall {v/ts*100:5.1f}%  inst {op_in[op]/ti*100:5.1f}%")
for d in sorted(data, reverse=True)[:n]: print(f"{d[0]/ts*100:5.1f}% {d[2]} {d[3][:90]}")

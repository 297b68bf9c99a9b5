"""SASS-level view of an ncu --page source CSV (--print-source cuda,sass): per instruction (address
order) the executed warp-instructions, stall samples and the two largest stall reasons.
usage: python tools/sass_view.py CSV [min_exec_fraction_of_max]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Address' in r][0]
hdr = rows[hi]
ai, si, ii = 2, hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
st = [(j, h) for j, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
wf = hdr.index('L1 Wavefronts Shared') if 'L1 Wavefronts Shared' in hdr else None
data = {}
cur = ''
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[0] == 'Line No':
        continue
    if r[0]:
        cur = r[0]
        continue
    if not r[ai].startswith('0x'):
        continue
    try:
        ex = float(r[ii]); sm = float(r[si])
    except ValueError:
        continue
    reasons = sorted(((float(r[j] or 0), h[6:]) for j, h in st), reverse=True)[:2]
    w = r[wf] if wf is not None else ''
    data[int(r[ai], 16)] = (cur, r[3].strip(), ex, sm, reasons, w)
mx = max(d[2] for d in data.values())
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
ts = sum(d[3] for d in data.values())
te = sum(d[2] for d in data.values())
print(f"total samples {ts:.0f}  warp-inst {te:.3e}")
for a in sorted(data):
    l, s, ex, sm, rs, w = data[a]
    if ex >= thr * mx or sm >= 0.005 * ts:
        rr = ' '.join(f"{n}:{v/ max(sm,1)*100:.0f}%" for v, n in rs if v > 0)
        print(f"{a & 0xfffff:05x} L{l:>4} ex{ex/mx:5.2f} st{sm/ts*100:5.1f}% wf{w:>6} {s[:60]:60s} {rr}")

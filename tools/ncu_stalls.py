"""Summarise warp-stall samples of an ncu source-page CSV (--page source --csv --print-source sass).
usage: python tools/ncu_stalls.py src.csv [window]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 64
hdr = rows[1]
rs = [r for r in rows[2:] if len(r) == len(hdr)]
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(int(r[2]) for r in rs)
print('total samples', tot)
agg = {hdr[i]: sum(int(r[i] or 0) for r in rs) for i in cols}
print('by reason:', sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
for w0 in range(0, len(rs), win):
    chunk = rs[w0:w0 + win]
    s = sum(int(r[2]) for r in chunk)
    if s < tot * 0.02:
        continue
    reasons = {hdr[i]: sum(int(r[i] or 0) for r in chunk) for i in cols}
    top = sorted(((v, k) for k, v in reasons.items() if v), reverse=True)[:4]
    ops = [r[1].strip().split()[0] if not r[1].strip().startswith('@') else r[1].strip().split()[1] for r in chunk]
    tags = sorted(set(o for o in ops if o.split('.')[0] in ('LDTM', 'UTCHMMA', 'LDGSTS', 'STS', 'UTMASTG', 'LDG', 'MUFU', 'SYNCS', 'UTMALDG', 'STG')))
    print(f"[{w0:5d}-{w0 + len(chunk):5d}] {s:7d} ({100 * s / tot:4.1f}%) {top} {tags[:6]}")

"""Aggregate an `ncu --page source --csv --print-source sass` export by SASS
region: share of executed instructions and of warp-stall samples per
window of instructions, plus the top instructions by samples.
Usage: python tools/sass_regions.py file.csv [window] [kernel index]"""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
sec = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # which kernel of a multi-kernel export
print(lines[starts[sec]][:120])
rows = list(csv.DictReader(lines[starts[sec] + 1:starts[sec + 1]]))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = lambda r, k: float(r[k] or 0)
ti = sum(f(r, 'Instructions Executed') for r in rows)
ts = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in rows)
print(f"{len(rows)} SASS instructions, {ti:.0f} warp instructions executed, {ts:.0f} samples")
for i in range(0, len(rows), win):
    ch = rows[i:i + win]
    ii = sum(f(r, 'Instructions Executed') for r in ch)
    ss = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in ch)
    if ii / ti > 0.01 or ss / ts > 0.01:
        ops = {}
        for r in ch:
            op = r['Source'].split()[0] if r['Source'].split() else '?'
            if op.startswith('@'):
                op = r['Source'].split()[1]
            ops[op.split('.')[0]] = ops.get(op.split('.')[0], 0) + f(r, 'Instructions Executed')
        top = sorted(ops.items(), key=lambda x: -x[1])[:5]
        print(f"{i:5d} inst {100 * ii / ti:5.1f}% samples {100 * ss / ts:5.1f}%  " + " ".join(f"{k}:{v / max(ii, 1) * 100:.0f}" for k, v in top))
print("top by samples:")
for r in sorted(rows, key=lambda r: -f(r, 'Warp Stall Sampling (All Samples)'))[:25]:
    print(f"  {100 * f(r, 'Warp Stall Sampling (All Samples)') / ts:4.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:70]}")

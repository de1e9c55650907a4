#!/bin/bash
# Per-kernel device times (ncu, serialised) of a command: name, grid, block, ns.
#   bash tools/ncu_times.sh <regex-filter> <command...>
F=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv "$@" 2>/dev/null | python3 -c "
import csv, sys, re, collections
rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); gi = h.index('Grid Size'); bi = h.index('Block Size')
agg = collections.OrderedDict()
for r in rows[1:]:
    if not re.search('$F', r[ki]): continue
    key = (r[ki][:70], r[gi], r[bi]); agg.setdefault(key, []).append(float(r[vi].replace(',', '')))
for (k, g, b), v in agg.items():
    v.sort(); print(f'{k:70s} grid={g:14s} blk={b:10s} n={len(v):3d} median={v[len(v)//2]/1e3:9.2f} us min={v[0]/1e3:9.2f}')
"

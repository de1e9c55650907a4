"""Summarise an LM_LU_TRACE timeline (stderr of tools/lu_trace.py)."""
import re
import sys

hi, lo = {}, {}
order = []
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/lutrace.txt"):
    m = re.match(r"LUTRACE (hi|lo) (.+?)\s+end\s+([\d.]+) us\s+\(\+\s*([\d.]+)\)", line)
    if not m:
        continue
    (hi if m.group(1) == "hi" else lo)[m.group(2).strip()] = float(m.group(3))
    if m.group(1) == "hi":
        order.append((m.group(2).strip(), float(m.group(4))))
cat = {}
for name, d in order:
    k = name.split(" ")[0] + (" " + name.split(" ")[1] if name.startswith(("inner", "chain", "outer", "next")) else "")
    cat[k] = cat.get(k, 0.0) + d
end = max(hi.values())
print(f"hi stream end {end / 1e3:.1f} ms; time by step kind:")
for k, v in sorted(cat.items(), key=lambda x: -x[1]):
    print(f"  {k:14s} {v / 1e3:7.2f} ms")

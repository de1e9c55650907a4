"""Markdown table of the round's bench lines (profiles/rNN/bench_config*.json)
for DESIGN.md section 6."""
import json
import pathlib
import sys

R = pathlib.Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01")
NAMES = {"1": "1 fused `2A + B%C - A/(1+|B|)` 4096²", "2": "2 trace, diag-scale ×2, 4096²",
         "3a": "3a A·B·C·v (3 GEMV) 4096²", "3b": "3b X·Y·Z (100×8000 chain)", "3c": "3c Aᵀ·A SYRK 16384×2048",
         "4a": "4a inv(A)·b 8192², 64 rhs (exact LU)", "4b": "4b 4096 × 64² solves", "5a": "5a 262144 instances f64",
         "5a-f32": "5a f32", "5b": "5b 32768² row-sharded, 1 GPU"}
print("| config | value | ms/step | dominant kernel: achieved / ceiling | DRAM traffic vs algorithmic | CPU ref (1 core) | e2e |")
print("|---|---|---|---|---|---|---|")
for c in ["1", "2", "3a", "3b", "3c", "4a", "4b", "5a", "5a-f32", "5b"]:
    f = R / f"bench_config{c}.json"
    if not f.exists():
        continue
    d = json.loads(f.read_text())
    r = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    unit = d["unit"]
    val = f"{d['value']:.4g} {unit}" + (f" ({d['tflops']:.3g} TF/s)" if d.get("tflops") and unit != "TFLOP/s" else "")
    roof = (f"{r['kernel']}: {r['achieved']:.4g} / {r['peak']:.4g} {r['unit']} = **{100 * r['frac']:.1f}%**"
            if r else "—")
    tr = r.get("traffic")
    traffic = f"{tr / 1e6:.0f} MB / {r['work_per_launch'] / 1e6:.0f} MB" if tr and r.get("unit") == "GB/s" else (
        f"{tr / 1e6:.0f} MB" if tr else "—")
    print(f"| {NAMES[c]} | {val} | {d['ms_per_step']:.4g} | {roof} | {traffic} | "
          f"{cpu.get('value', 0):.3g} {unit} | {e2e.get('value', 0):.3g} {unit} |")

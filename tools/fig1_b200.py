"""The paper's Fig. 1 (naive vs optimised evaluation of the ten expressions,
PAPER.md:452-607) on a B200, through the public harness (harness.run_bench:
verify-before-time, mean of `runs` synchronised evaluations, lazymat/bench.py
methodology) -- SURVEY.md 8(f)3.

    python tools/fig1_b200.py [runs] > profiles/r02/fig1_b200.md
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2502_03000_b200.harness import report, run_bench  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
sizes = [100, 250, 500, 1000]
big = [2000, 4000]  # beyond the paper's sizes: where the device work outgrows the per-call host cost
# the reference package's acceptance bars at 500^2 (tests/test_acceptance.py:143-144)
BARS = {1: 30, 3: 80, 4: 80, 5: 95, 6: 25, 7: 95, 8: 20, 9: 40, 10: 80}
# Armadillo + OpenBLAS on a Ryzen 7640U at 1000^2, context only
PAPER_1000 = {1: 67.90, 3: 96.40, 5: 99.99, 6: 50.17, 8: 48.89, 9: 64.34}
recs = run_bench(range(1, 11), sizes, runs, 42, "both") + run_bench(range(1, 11), big, max(runs // 5, 3), 42, "both")
recs.sort(key=lambda r: (r.expr_id, r.size, r.mode))
print(f"# Fig. 1 on B200 ({torch.cuda.get_device_name(0)}), mean of {runs} synchronised evaluations "
      f"({max(runs // 5, 3)} at 2000 and 4000)\n")
print("Produced by `tools/fig1_b200.py` through `paper_2502_03000_b200.harness.run_bench` (the reference's "
      "methodology: verify naive vs optimised <= 1e-8 first, then time each arm). Seeded U[0,1) operands as in "
      "lazymat/bench.py:76-130; both arms run on the GPU (the naive arm materialises every node, inverts "
      "explicitly and multiplies chains left to right). A timed evaluation includes validation, the rewrite "
      "(planner, Python) and the launches: at the paper's sizes (<= 1000) both arms cost tens of microseconds "
      "of host work per call and the device work is a few microseconds, so the reductions there measure the "
      "planner's host cost, not the kernels; 2000 and 4000 show the regime where the device work dominates.\n")
print(report(recs, "markdown"))
by = {(r.expr_id, r.size, r.mode): r.mean_seconds for r in recs}
print("## Reductions at 500^2 against the reference package's acceptance bars, and at 1000^2 against the paper\n")
print("| expr | B200 reduction 500^2 | reference bar (500^2) | B200 reduction 1000^2 | paper (CPU, 1000^2) |")
print("| ---: | ---: | ---: | ---: | ---: |")
for e in range(1, 11):
    r5 = 100 * (1 - by[(e, 500, "optimised")] / by[(e, 500, "naive")])
    r10 = 100 * (1 - by[(e, 1000, "optimised")] / by[(e, 1000, "naive")])
    bar = BARS.get(e)
    ok = "" if bar is None else (" (meets)" if r5 >= bar else " (below)")
    print(f"| ({e}) | {r5:.2f}%{ok} | {f'>= {bar}%' if bar else '-'} | {r10:.2f}% | "
          f"{f'{PAPER_1000[e]:.2f}%' if e in PAPER_1000 else '-'} |")
print("\n## CSV\n\n```\n" + report(recs, "csv") + "\n```")

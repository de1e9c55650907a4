"""Golden for the seeded random-tree fuzz (tests/golden/fuzz_trees.py):
the REFERENCE's render_expr text and validate() result -- shape, or error
type and message -- for 400 trees.  Build container only.

    python tests/golden/make_golden_fuzz.py
"""

import json
import os
import pathlib
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lm_numba_cache"))
sys.dont_write_bytecode = True
HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import lazymat  # noqa: E402
from fuzz_trees import record, trees, value_record  # noqa: E402

if __name__ == "__main__":
    rec = record(lazymat)
    vals = [value_record(lazymat, t) if r[1][0] == "ok" else None for t, r in zip(trees(lazymat), rec)]
    (HERE / "fuzz_trees.json").write_text(json.dumps({"trees": rec, "values": vals}, indent=0))
    print("wrote", len(rec), "trees;", sum(r[1][0] == "error" for r in rec), "errors;",
          sum(1 for v in vals if v and v[0] == "error"), "evaluation errors")

"""Regenerate only the `adapter` section of golden.json (the whole-program
adapter's per-construct records), leaving every other fixture untouched.
Needs the reference (/root/reference) — run in the build container:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/update_adapter.py
"""
import json
import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import make_golden as M  # noqa: E402

if __name__ == "__main__":
    path = HERE / "golden.json"
    g = json.loads(path.read_text())
    from corpus import CORPUS
    g["adapter"] = M.record_adapter_constructs(CORPUS)
    path.write_text(json.dumps(g, indent=1, sort_keys=True))
    n = sum(len(v["constructs"]) for v in g["adapter"].values())
    print(f"adapter records: {n}")

"""Print the structural signatures of the case-study accelerated bindings
(paper_2211_00621_b200/dropin_programs.py SIGNATURES) from the programs in
tests/golden/golden.json, running the reference (baseline/_ref or
/root/reference) with a hook on pmx.interp.device_call.

    python tools/dropin_signatures.py
"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
for p in (ROOT / "baseline" / "_ref", pathlib.Path("/root/reference/pkg/src")):
    if (p / "pmx").exists():
        sys.path.insert(0, str(p))
        break

import pmx  # noqa: E402
import pmx.interp as interp  # noqa: E402
import pmx.runtime as rt  # noqa: E402
import pmx.syntax as syn  # noqa: E402
from paper_2211_00621_b200 import dropin_programs as D  # noqa: E402

G = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
progs = [("program_rk4", G["program_rk4"]["program"]), ("program_viterbi", G["program_viterbi"]["program"]),
         ("program_nn", G["program_nn"]["program"])]
for sec in ("rk4_param", "hmm_forward", "knn", "kmer"):
    for i, e in enumerate(G[sec]):
        progs.append((f"{sec}/{i}", e["program"]))

orig = interp.device_call
seen = []


def hook(fn, args, ctx, span):
    c = D.canon(fn, syn, rt)
    seen.append((c, fn, args))
    return orig(fn, args, ctx, span)


interp.device_call = hook
for name, src in progs:
    seen.clear()
    pmx.run_source(src, mode="accel", workers=2, capture_output=True)
    for c, fn, args in seen:
        caps = [(n, type(v).__name__ + (f"[{len(v)}]" if isinstance(v, list) else f"={v!r}")) for n, v in c.caps]
        print(f"{name:18s} {c.digest()}  params={[p.text for p in fn.params]} "
              f"args={[type(a).__name__ + (f'[{len(a)}]' if isinstance(a, list) else '') for a in args]}")
        print(f"{'':18s} caps={caps}")
        print(f"{'':18s} lits={c.lits}")

"""Generate tests/golden/golden.json by running the REFERENCE interpreter.

Run in the container that has /root/reference (the GPU box does not):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is the stdout (or RuntimeError message) of a PMExpr program
executed by `pmx.run_source`, so the expected values are the reference's own
answers.  Programs are stored next to their outputs.  The oracle (oracle/)
is pinned against these fixtures (tests/test_oracle.py) and the B200 path is
checked against both (tests/test_gpu_*.py).
"""
from __future__ import annotations

import json
import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(HERE.parent.parent))
sys.setrecursionlimit(100_000)

from pmx import Diagnostics, run_source  # noqa: E402

import cases  # noqa: E402  (tests/golden/cases.py)


def run(src: str, mode: str = "debug", workers: int = 1) -> dict:
    try:
        r = run_source(src, mode=mode, workers=workers, capture_output=True)
        return {"stdout": r.stdout}
    except Diagnostics as d:
        return {"error": "\n".join(x.message for x in d.items)}


def lit(v) -> str:
    if isinstance(v, float):
        return repr(v)
    return str(v)


def seq_lit(vs) -> str:
    return "[" + ", ".join(lit(v) for v in vs) + "]"


def print_each(var: str, conv: str) -> str:
    return f'foldl (lam u. lam x. let p = print ({conv} x) in print " ") {{}} {var}'


def map_case(pm_lambda: str, inputs) -> dict:
    for conv in ("int2string", "float2string"):
        src = (f"let s = {seq_lit(inputs)} in\nlet f = lam xs. map ({pm_lambda}) xs in\n"
               f"let r = accelerate (f s) in\n{print_each('r', conv)}\n")
        try:
            from pmx import compile_source
            compile_source(src)
        except Diagnostics:
            continue
        out = run(src, mode="accel", workers=4)
        out["program"] = src
        out["conv"] = conv
        return out
    raise RuntimeError(f"no printer for {pm_lambda}")


def scalar_prog(body: str, inputs, conv_candidates=("int2string", "float2string")) -> dict:
    from pmx import compile_source
    s = seq_lit(inputs) if inputs else "create 0 (lam i. i)"
    for conv in conv_candidates:
        src = f"let s = {s} in\nlet f = lam xs. {body} in\nlet r = accelerate (f s) in\nprint ({conv} r)\n"
        try:
            compile_source(src)
        except Diagnostics:
            continue
        out = run(src, mode="accel", workers=4)
        out["program"] = src
        return out
    raise RuntimeError(body)


H = "(lam a. lam m. divi (modi (muli a m) 4294967296) 65536)"

HMM_FWD = """
let numStates = {S} in
let numSymbols = {K} in
let numSignals = {NS} in
let obsLen = {T} in
let rowNorm = lam row. let total = foldl addf 0.0 row in map (lam p. divf p total) row in
let transition = create numStates (lam i. rowNorm (create numStates (lam j.
    int2float (addi 1 (modi (addi (addi (muli i 131) (muli j 71)) (muli (muli i j) 7)) 97))))) in
let emission = create numStates (lam j. rowNorm (create numSymbols (lam k.
    int2float (addi 1 (modi (addi (addi (muli j 13) (muli k 29)) (muli (muli j k) 3)) 31))))) in
let initial = rowNorm (create numStates (lam i. int2float (addi 1 (modi i 17)))) in
let h = {H} in
let signals = create numSignals (lam s. create obsLen (lam t.
    modi (h (addi (muli s obsLen) t) 2654435761) numSymbols)) in
let forwardAll = lam trans. lam emit. lam init. lam sigs.
  let logTrans = create numStates (lam i. create numStates (lam j. log (get (get trans i) j))) in
  let logEmit = create numStates (lam i. create numSymbols (lam k. log (get (get emit i) k))) in
  let lse = lam xs.
    let m = foldl (lam a. lam x. match gtf x a with true then x else a) (get xs 0) xs in
    addf m (log (foldl (lam a. lam x. addf a (exp (subf x m))) 0.0 xs)) in
  let one = lam obs.
    let n = length obs in
    let a0 = create numStates (lam i. addf (log (get init i)) (get (get logEmit i) (get obs 0))) in
    recursive let go = lam t. lam alpha.
      match eqi t n with true then alpha else
      go (addi t 1) (create numStates (lam j.
        addf (lse (create numStates (lam i. addf (get alpha i) (get (get logTrans i) j))))
             (get (get logEmit j) (get obs t))))
    in lse (go 1 a0)
  in map one sigs
in
let ll = accelerate (forwardAll transition emission initial signals) in
foldl (lam u. lam x. let p = print (float2string x) in print " ") {{}} ll
"""

KNN = """
let numTrain = {NT} in
let numQuery = {NQ} in
let dim = {D} in
let k = {KK} in
let numClasses = {C} in
let dimIdx = create dim (lam i. i) in
let classIdx = create numClasses (lam c. c) in
let h = {H} in
let train = create numTrain (lam p. create dim (lam i.
    int2float (subi (modi (h (addi (muli p dim) i) 2654435761) 17) 8))) in
let labels = create numTrain (lam p. modi (divi (modi (muli p 2654435761) 4294967296) 1048576) numClasses) in
let queries = create numQuery (lam q. create dim (lam i.
    int2float (subi (modi (h (addi (muli q dim) i) 2246822519) 17) 8))) in
let classify = lam tr. lam lab. lam qs.
  let dist = lam a. lam b. foldl (lam acc. lam i.
      let d = subf (get a i) (get b i) in addf acc (mulf d d)) 0.0 dimIdx in
  let better = lam d1. lam i1. lam d2. lam i2.
      match ltf d1 d2 with true then true else match eqf d1 d2 with true then lti i1 i2 else false in
  recursive let ins = lam lst. lam d. lam i. lam pos.
      match eqi pos k with true then lst else
      let c = get lst pos in
      match better d i c.d c.i with true then
        ins (set lst pos {{d = d, i = i}}) c.d c.i (addi pos 1)
      else ins lst d i (addi pos 1)
  in
  let one = lam q.
    let init = create k (lam j. {{d = 1.0e308, i = 9223372036854775807}}) in
    let top = foldl (lam lst. lam p. ins lst (dist q (get tr p)) p 0) init (create numTrain (lam p. p)) in
    let votes = create numClasses (lam c. foldl (lam acc. lam e.
        match eqi (get lab e.i) c with true then addi acc 1 else acc) 0 top) in
    foldl (lam best. lam c. match gti (get votes c) (get votes best) with true then c else best) 0 classIdx
  in map one qs
in
let preds = accelerate (classify train labels queries) in
foldl (lam u. lam x. let p = print (int2string x) in print " ") {{}} preds
"""

KMER = """
let kmer = {KM} in
let numStates = {S} in
let hi = {HI} in
let numSymbols = {K} in
let numSignals = {NS} in
let obsLen = {T} in
let rowNorm = lam row. let total = foldl addf 0.0 row in map (lam p. divf p total) row in
let emission = create numStates (lam j. rowNorm (create numSymbols (lam k.
    int2float (addi 1 (modi (addi (addi (muli j 13) (muli k 29)) (muli (muli j k) 3)) 31))))) in
let h = {H} in
let signals = create numSignals (lam s. create obsLen (lam t.
    modi (h (addi (muli s obsLen) t) 2654435761) numSymbols)) in
let forwardAll = lam emit. lam sigs.
  let logEmit = create numStates (lam i. create numSymbols (lam k. log (get (get emit i) k))) in
  let lstay = log {PSTAY} in
  let lstep = log {PSTEP} in
  let l0 = log (divf 1.0 (int2float numStates)) in
  let lse = lam xs.
    let m = foldl (lam a. lam x. match gtf x a with true then x else a) (get xs 0) xs in
    addf m (log (foldl (lam a. lam x. addf a (exp (subf x m))) 0.0 xs)) in
  let one = lam obs.
    let n = length obs in
    let a0 = create numStates (lam i. addf l0 (get (get logEmit i) (get obs 0))) in
    recursive let go = lam t. lam alpha.
      match eqi t n with true then alpha else
      go (addi t 1) (create numStates (lam j.
        let base = divi j 4 in
        addf (lse [addf (get alpha j) lstay,
                   addf (get alpha base) lstep,
                   addf (get alpha (addi base hi)) lstep,
                   addf (get alpha (addi base (muli 2 hi))) lstep,
                   addf (get alpha (addi base (muli 3 hi))) lstep])
             (get (get logEmit j) (get obs t))))
    in lse (go 1 a0)
  in map one sigs
in
let ll = accelerate (forwardAll emission signals) in
foldl (lam u. lam x. let p = print (float2string x) in print " ") {{}} ll
"""

MAPREDUCE = """
let n = {N} in
let s = create n (lam i. divf (int2float (divi (modi (muli i 2654435761) 4294967296) 1024)) 4194304.0) in
let f = lam xs. reduce addf 0.0 (map (lam x. addf (mulf 2.0 x) 1.0) xs) in
let r = accelerate (f s) in
print (float2string r)
"""

RK4_PARAM = """
let numParams = {N} in
let numSteps = {M} in
let h = 0.01 in
let dims = create 4 (lam i. i) in
let params = create numParams (lam k. addf 0.5 (divf (int2float k) (int2float numParams))) in
"""


def rk4_variant(n: int, m: int) -> str:
    src = (REF / "programs" / "rk4.pmx").read_text()
    head_end = src.index("let deriv")   # replaces numParams/numSteps/h/dims/params
    return RK4_PARAM.format(N=n, M=m) + src[head_end:]


def main() -> None:
    g: dict = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg (pmx)"}
    g["map"] = {name: dict(map_case(pm, xs), type=ty, inputs=xs) for name, pm, _, ty, xs in cases.MAP_CASES}
    g["reduce"] = {name: dict(scalar_prog(f"reduce ({op}) {acc} xs", xs), type=ty, inputs=xs, acc=accv)
                   for name, op, _, acc, accv, ty, xs in cases.REDUCE_CASES}
    g["foldl"] = {name: dict(scalar_prog(f"foldl ({op}) {acc} (map (lam x. x) xs)", xs), type=ty, inputs=xs, acc=accv)
                  for name, op, _, acc, accv, ty, xs in cases.FOLD_CASES}
    g["map2"] = {}
    for name, op, _, ty, xs, ys in cases.MAP2_CASES:
        conv = "float2string" if ty == "float" else "int2string"
        src = (f"let a = {seq_lit(xs)} in\nlet b = {seq_lit(ys)} in\nlet f = lam p. lam q. map2 ({op}) p q in\n"
               f"let r = accelerate (f a b) in\n{print_each('r', conv)}\n")
        g["map2"][name] = dict(run(src, mode="accel", workers=4), program=src, type=ty, x=xs, y=ys)

    from corpus import CORPUS
    g["corpus"] = {name: dict(run(src), program=src, float_rel=rel) for name, src, rel in CORPUS}

    from test_interp import ACCEL_SUM
    from test_acceptance import ALIAS_PROGRAM
    g["accel_sum"] = {str(w): run(ACCEL_SUM, mode="accel", workers=w) for w in (1, 2, 3, 8, 16)}
    g["accel_sum"]["program"] = ACCEL_SUM
    g["alias"] = {str(w): run(ALIAS_PROGRAM, mode="accel", workers=w) for w in (1, 2, 8)}
    g["alias"]["program"] = ALIAS_PROGRAM

    for prog in ("rk4", "viterbi", "nn"):
        src = (REF / "programs" / f"{prog}.pmx").read_text()
        g[f"program_{prog}"] = dict(run(src, mode="accel", workers=4), program=src)

    g["rk4_param"] = []
    for n, m in ((6, 60), (3, 200)):
        src = rk4_variant(n, m)
        g["rk4_param"].append(dict(run(src, mode="accel", workers=4), N=n, M=m, program=src))

    g["hmm_forward"] = []
    for S, K, NS, T in ((4, 8, 3, 12), (8, 8, 2, 16), (16, 4, 2, 8)):
        src = HMM_FWD.format(S=S, K=K, NS=NS, T=T, H=H)
        g["hmm_forward"].append(dict(run(src, mode="accel", workers=4), S=S, K=K, NS=NS, T=T, program=src))

    g["knn"] = []
    for NT, NQ, D, KK, C in ((60, 8, 8, 3, 4), (100, 6, 16, 8, 10), (40, 5, 4, 1, 3)):
        src = KNN.format(NT=NT, NQ=NQ, D=D, KK=KK, C=C, H=H)
        g["knn"].append(dict(run(src, mode="accel", workers=4), NT=NT, NQ=NQ, D=D, K=KK, C=C, program=src))

    g["kmer"] = []
    for KM, K, NS, T in ((2, 4, 2, 8), (3, 8, 2, 5)):
        S = 1 << (2 * KM)
        src = KMER.format(KM=KM, S=S, HI=1 << (2 * KM - 2), K=K, NS=NS, T=T, H=H, PSTAY="0.5", PSTEP="0.125")
        g["kmer"].append(dict(run(src, mode="accel", workers=4), kmer=KM, K=K, NS=NS, T=T,
                              p_stay=0.5, p_step=0.125, program=src))

    g["mapreduce"] = []
    for N, W in ((4096, 4), (1000, 3)):
        src = MAPREDUCE.format(N=N)
        g["mapreduce"].append(dict(run(src, mode="accel", workers=W), N=N, workers=W, program=src))

    g["adapter"] = record_adapter_constructs(CORPUS)

    out = HERE / "golden.json"
    out.write_text(json.dumps(g, indent=1, sort_keys=True))


def record_adapter_constructs(corpus) -> dict:
    """Run every corpus program in accel mode with the reference's own
    skeletons, and for each device-context construct record the adapter's
    translation of its function argument (lambda IR as JSON, with captured
    host data), its inputs and the reference's result.  tests/test_gpu_adapter.py
    replays each construct on the B200."""
    import pmx.interp as interp
    import pmx.runtime as rt
    import pmx.syntax as syn
    from paper_2211_00621_b200 import ir_json, pmx_adapter

    orig = {n: getattr(interp, n) for n in ("eval_map", "eval_map2", "eval_reduce", "eval_loop")}
    records: list = []

    def conv(s):
        return [ord(x) if isinstance(x, str) else (dict(x) if isinstance(x, dict) else x) for x in s]

    def elem(s):
        x = s[0] if s else 0
        return "char" if isinstance(x, str) else ("bool" if isinstance(x, bool) else
                                                  ("float" if isinstance(x, float) else
                                                   ("record" if isinstance(x, dict) else "int")))

    def translate(f, n, ctx, tensors):
        def host_array(v):
            if isinstance(v, rt.TensorView):
                buf = ctx.heap.buffers[v.buffer]
                h = ir_json.HostArray(list(buf), v.elem, v.shape, v.offset)
                tensors.append((h, buf))
                return h
            return ir_json.HostArray(conv(v), elem(v))
        try:
            return ir_json.dump(pmx_adapter.to_lam(f, n, syn, rt, host_array))
        except pmx_adapter.Unsupported:
            return None

    def rec(kind, ctx, f, arity, call, **kw):
        tensors: list = []
        lam = translate(f, arity, ctx, tensors) if ctx.run_parallel else None
        out = call()
        if lam is not None:
            r = dict(kind=kind, lam=lam, expected=out if kind != "loop" else None, **kw)
            if kind == "loop":
                r["tensors_after"] = [list(buf) for _, buf in tensors]
            records.append(r)
        return out

    def eval_map(f, s, ctx, span):
        if s and isinstance(s[0], list):              # row function over [[a]]
            out = orig["eval_map"](f, s, ctx, span)
            if ctx.run_parallel:
                tensors: list = []
                try:
                    g, op, acc = pmx_adapter.to_row_fold(f, syn, rt, lambda v: ir_json.HostArray(conv(v), elem(v)))
                    records.append(dict(kind="map_rows", g=ir_json.dump(g) if g is not None else None,
                                        op=ir_json.dump(op), acc=acc, rows=[conv(r) for r in s],
                                        x_elem=elem(s[0]), expected=out))
                except pmx_adapter.Unsupported:
                    pass
            return out
        return rec("map", ctx, f, 1, lambda: orig["eval_map"](f, s, ctx, span), xs=conv(s), x_elem=elem(s)) \
            if s else orig["eval_map"](f, s, ctx, span)

    def eval_map2(f, s1, s2, ctx, span):
        return rec("map2", ctx, f, 2, lambda: orig["eval_map2"](f, s1, s2, ctx, span), xs=conv(s1), ys=conv(s2),
                   x_elem=elem(s1), y_elem=elem(s2)) if s1 else orig["eval_map2"](f, s1, s2, ctx, span)

    def eval_reduce(f, acc, s, ctx, span):
        return rec("reduce", ctx, f, 2, lambda: orig["eval_reduce"](f, acc, s, ctx, span), acc=acc, xs=conv(s),
                   x_elem=elem(s)) if s else orig["eval_reduce"](f, acc, s, ctx, span)

    def eval_loop(n, f, ctx, span):
        return rec("loop", ctx, f, 1, lambda: orig["eval_loop"](n, f, ctx, span), n=n) \
            if n > 0 else orig["eval_loop"](n, f, ctx, span)

    out: dict = {}
    interp.eval_map, interp.eval_map2, interp.eval_reduce, interp.eval_loop = eval_map, eval_map2, eval_reduce, eval_loop
    try:
        for name, src, rel in corpus:
            records.clear()
            try:
                run_source(src, mode="accel", workers=4, capture_output=True)
            except Diagnostics:
                pass
            out[name] = {"float_rel": rel, "constructs": list(records)}
    finally:
        for k, v in orig.items():
            setattr(interp, k, v)
    return out
    print(f"wrote {out}")


if __name__ == "__main__":
    main()

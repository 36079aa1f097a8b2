"""The whole-program drop-in on the B200.

The reference package, installed unmodified in baseline/_ref,
has its skeletons and `device_call` replaced by pmx_adapter.install(); every
program of the golden fixtures then runs through the reference's own
`pmx.run_source(mode="accel")`: its parser, type checker, accelerate
rewrite, lifting and interpreter on the host, every accelerated construct on
the B200.  Output must match the reference's (tests/test_acceptance.py:246-253:
debug-mode stdout, tokens compared with the corpus tolerance).
tests/golden/golden.json carries each program's source and the reference's
output (tests/golden/make_golden.py)."""
import pathlib
import sys

import pytest

from conftest import GOLDEN, tokens_match

REF = pathlib.Path(__file__).resolve().parent.parent / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "pmx").exists(), reason="baseline/_ref (the reference) not installed")]


def _programs():
    out = []
    for name, e in sorted(GOLDEN["corpus"].items()):
        out.append((f"corpus/{name}", e["program"], e, e.get("float_rel") or 1e-12, 4))
    for w in ("1", "2", "3", "8", "16"):
        out.append((f"accel_sum/w{w}", GOLDEN["accel_sum"]["program"], GOLDEN["accel_sum"][w], 1e-12, int(w)))
    for w in ("1", "2", "8"):
        out.append((f"alias/w{w}", GOLDEN["alias"]["program"], GOLDEN["alias"][w], 1e-12, int(w)))
    for sec in ("map2",):
        for name, e in sorted(GOLDEN[sec].items()):
            out.append((f"{sec}/{name}", e["program"], e, 1e-12, 4))
    for sec, rel in (("mapreduce", 1e-12), ("hmm_forward", 1e-5), ("knn", 0.0), ("kmer", 1e-5),
                     ("rk4_param", 1e-9)):
        for i, e in enumerate(GOLDEN[sec]):
            out.append((f"{sec}/{i}", e["program"], e, rel, 4))
    for prog, rel in (("rk4", 1e-9), ("viterbi", 1e-9), ("nn", 1e-9)):
        e = GOLDEN[f"program_{prog}"]
        out.append((f"programs/{prog}.pmx", e["program"], e, rel, 4))
    return out


PROGRAMS = _programs() if (REF / "pmx").exists() else []
FAMILY = {"programs/rk4.pmx": "rk4", "programs/viterbi.pmx": "viterbi", "programs/nn.pmx": "nn",
          "rk4_param": "rk4", "hmm_forward": "hmm_forward", "knn": "knn", "kmer": "hmm_kmer"}


@pytest.fixture(scope="module")
def pmx_installed():
    sys.path.insert(0, str(REF))
    import pmx
    import pmx.interp as interp
    from paper_2211_00621_b200 import pmx_adapter
    uninstall = pmx_adapter.install(interp)
    yield pmx, pmx_adapter
    uninstall()


@pytest.mark.parametrize("name,src,want,rel,workers", PROGRAMS, ids=[p[0] for p in PROGRAMS])
def test_program_through_the_b200_dropin(pmx_installed, name, src, want, rel, workers):
    pmx, adapter = pmx_installed
    if "error" in want:
        with pytest.raises(pmx.Diagnostics) as ei:
            pmx.run_source(src, mode="accel", workers=workers, capture_output=True)
        assert want["error"] in str(ei.value)
        return
    out = pmx.run_source(src, mode="accel", workers=workers, capture_output=True).stdout
    assert tokens_match(out, want["stdout"], float_rel=rel), (out[:400], want["stdout"][:400])
    family = FAMILY.get(name.split("/")[0] if not name.startswith("programs/") else name)
    if family is not None:          # ran as its case-study kernel, not construct by construct
        assert adapter.install.last_binding == family


def test_one_upload_per_accelerate_call(pmx_installed):
    # a sequence used by two constructs of one accelerate call crosses to the
    # device once; the map's result feeds the reduce from the device
    pmx, adapter = pmx_installed
    src = ("let f = lam s. let a = map (lam x. muli x 3) s in let b = map (lam x. addi x 1) s in "
           "reduce addi 0 (map2 (lam p. lam q. addi p q) a b) in "
           "let r = accelerate (f [1, 2, 3, 4, 5]) in print (int2string r)")
    out = pmx.run_source(src, mode="accel", workers=2, capture_output=True).stdout
    assert out == str(sum(3 * x + x + 1 for x in range(1, 6)))
    call = adapter.install.last_call
    assert call is not None and call.h2d_sequences == 1


def test_read_only_tensor_is_not_copied_back(pmx_installed):
    # the alias program writes one tensor view and reads another: only the
    # written buffer's device mirror is copied back after the loop
    pmx, adapter = pmx_installed
    out = pmx.run_source(GOLDEN["alias"]["program"], mode="accel", workers=2, capture_output=True).stdout
    assert out == "7"
    call = adapter.install.last_call
    assert all(m.uploads == 1 for m in call.mirrors.values())


def test_check_determinism_warns_like_the_reference(pmx_installed, capsys):
    # a non-associative operator (subtraction): the device tree and the
    # element-order re-fold differ, and the reference's warning is printed
    pmx, _ = pmx_installed
    src = ("let f = lam s. reduce (lam a. lam b. subf a b) 0.0 s in "
           "let r = accelerate (f (create 4096 (lam i. int2float (modi (muli i 7) 13)))) in "
           "print (float2string r)")
    pmx.run_source(src, mode="accel", workers=4, check_determinism=True, capture_output=True)
    err = capsys.readouterr().err
    assert "warning: reduce result depends on the evaluation order" in err


KTERM = [
    ("recursive let fib = lam n. match n with 0 then 0 else match n with 1 then 1 else "
     "addi (fib (subi n 1)) (fib (subi n 2)) in "
     "let r = accelerate (map fib [0, 1, 2, 3, 7, 15]) in print (int2string (reduce addi 0 r))"),
    ("recursive let t = lam n. match n with 3 then 1 else match n with 1 then 0 else "
     "match n with 2 then 0 else addi (t (subi n 3)) (addi (t (subi n 1)) (t (subi n 2))) in "
     "let r = accelerate (map t [1, 2, 3, 4, 10, 13]) in print (int2string (reduce addi 0 r))"),
    ("recursive let g = lam x. lam n. match n with 0 then x else match n with 1 then 1.0 else "
     "let a = g x (subi n 1) in let b = g x (subi n 2) in addf (mulf 0.5 a) (mulf x b) in "
     "let r = accelerate (map (lam n. g 0.25 n) [0, 1, 2, 9, 14]) in print (float2string (reduce addf 0.0 r))"),
]


@pytest.mark.parametrize("src", KTERM, ids=["fib", "tribonacci", "kterm_float"])
def test_kterm_recursion_through_the_dropin(pmx_installed, src):
    # non-linear (k-term) recursion runs as a device loop with k accumulators;
    # the reference's own debug mode is the expected output
    pmx, _ = pmx_installed
    want = pmx.run_source(src, mode="debug", capture_output=True).stdout
    got = pmx.run_source(src, mode="accel", workers=4, capture_output=True).stdout
    assert tokens_match(got, want, float_rel=1e-12), (got, want)


def test_kterm_recursion_at_specialised_kernel_size(pmx_installed):
    # 70,000 elements: the map runs in the run-time specialised kernel (above
    # the interpreter threshold); expected value from the closed iteration
    pmx, _ = pmx_installed
    src = ("recursive let fib = lam n. match n with 0 then 0 else match n with 1 then 1 else "
           "addi (fib (subi n 1)) (fib (subi n 2)) in "
           "let r = accelerate (map fib (create 70000 (lam i. modi i 45))) in print (int2string (reduce addi 0 r))")
    f = [0, 1]
    while len(f) < 45:
        f.append(f[-1] + f[-2])
    want = sum(f[i % 45] for i in range(70000))
    got = pmx.run_source(src, mode="accel", workers=4, capture_output=True).stdout
    assert int(got) == want

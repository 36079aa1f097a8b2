"""Benchmark of the accelerated-expression hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload mapreduce|rk4|knn|hmm|kmer] [--no-case-studies]

Headline workload (BASELINE.json configs[1]): the map/reduce skeleton
microbench — `reduce addf 0.0 (map (lam x. addf (mulf 2.0 x) 1.0) s)` over
2^28 fp32 elements per GPU (weak scaling: every rank owns 2^28 elements of
an N*2^28-element sequence, partitioned like _chunks, pmx/interp.py:273-276;
the per-GPU partials are combined with one NCCL all-gather and a fixed-order
fold on the device).  One step = one evaluation of that expression.  Inputs
(1 GiB per GPU) are larger than L2 (126 MB), so no flush is needed.

`value` is device-resident throughput (elements/s, all ranks), `e2e` the same
program through the public `accelerate` entry with pinned HOST input (H2D of
the input + kernel + D2H of the result inside the timed region).  The case
studies (RK4, k-NN, HMM forward, k-mer HMM) are reported under
`case_studies` with their own roofline and CPU-oracle baselines.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "elements/s per case study (HMM, k-NN, RK4) at 1/2/4/8 B200 vs CPU ref"
N_PER_GPU = 1 << 28


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


# ------------------------------------------------------------- distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend: str):
        # PMX_DIST_BACKEND=gloo: exercise the N>1 code path with several ranks
        # sharing one GPU (functional check only — no meaningful timing)
        import torch.distributed as dist
        self.backend = os.environ.get("PMX_DIST_BACKEND", backend)
        if self.world > 1 and not dist.is_initialized():
            dist.init_process_group(self.backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def all_gather(self, out, t):
        """all_gather_into_tensor (NCCL) or its CPU equivalent (gloo)."""
        if self.backend == "nccl":
            self.pg.all_gather_into_tensor(out, t)
            return
        parts = [torch_cpu_like(t) for _ in range(self.world)]
        self.pg.all_gather(parts, t.cpu())
        out.copy_(__import__("torch").cat(parts).to(out.device))

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())


def torch_cpu_like(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype)


# ------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi samples during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = []
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:]) if v.lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- timing
def device_time(step, steps: int, warmup: int, dist: Dist, per_step_events: bool = True):
    """W untimed steps, then EXACTLY K steps between barrier+synchronize on
    both sides, timed with CUDA events on the launching stream; returns
    (total ms max over ranks, list of per-step ms on this rank)."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(st)
    for i in range(steps):
        step()
        evs[i + 1].record(st)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    total = evs[0].elapsed_time(evs[-1])
    return dist.max(total), per


def host_time(step, steps: int, warmup: int, dist: Dist):
    """End-to-end: each step ends with a host read of its result, so host
    wall time between synchronised points equals device-stream time."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dist.barrier()
    return dist.max(e0.elapsed_time(e1)), (t1 - t0) * 1e3


def cpu_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


# ============================================================ map/reduce
def bench_mapreduce(args, dist: Dist, peaks: dict) -> dict:
    import numpy as np
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib, synth
    from paper_2211_00621_b200.runtime import DeviceSeq
    from paper_2211_00621_b200.skeletons import default_ctx, PreparedMapReduce

    n = N_PER_GPU
    dev = torch.device("cuda", torch.cuda.current_device())
    f = P.lam("x", P.addf(P.mulf(2.0, "x"), 1.0))
    # rank r owns elements [r*n, (r+1)*n) of the global sequence (_chunks rule)
    x = synth.mapreduce_x_device(n * dist.world, dev)[dist.rank * n:(dist.rank + 1) * n].contiguous() \
        if dist.world > 1 else synth.mapreduce_x_device(n, dev)
    seq = DeviceSeq(x, (n,), _lib.PMX_F32)
    ctx = default_ctx()
    prep = PreparedMapReduce(f, P.addf, 0.0, seq, ctx)
    gathered = torch.empty(dist.world, dtype=torch.float64, device=dev)

    def combine(partial):
        if dist.world == 1:
            return partial
        dist.all_gather(gathered, partial)
        return prep.fold_partials(gathered)           # fixed rank order (interp.py:334-336)

    # N > 1: the shard partials are exchanged over NVLink peer memory by the
    # reduce kernel itself (one launch per step, no collective); the NCCL
    # all-gather + fold path is timed beside it as a variant.
    peers = None
    if dist.world > 1 and not args.nccl_combine:
        from paper_2211_00621_b200.shard import PeerMailboxes
        peers = PeerMailboxes()

    def step():
        if peers is not None:
            prep.launch_peers(peers)
        else:
            combine(prep.launch())

    launches0 = ctx.launches
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    total_ms, per = device_time(step, args.steps, args.warmup, dist)
    clk = clocks.stop()
    launches = (ctx.launches - launches0) // (args.steps + args.warmup) * args.steps
    result = float((prep.launch_peers(peers) if peers is not None else combine(prep.launch())).item())
    nccl_ms = None
    if dist.world > 1:
        nccl_ms, _ = device_time(lambda: combine(prep.launch()), args.steps, 1, dist)
    ctx.check_errors()
    exact = synth.mapreduce_exact_sum(n) if dist.world == 1 else None

    # variants: the individual skeleton kernels (map only 8 B/elem, reduce only 4 B/elem)
    y = torch.empty_like(x)
    prep_map = PreparedMapReduce(f, P.addf, 0.0, seq, ctx, materialize=y, reduce=False)
    map_ms, _ = device_time(prep_map.launch, args.steps, 1, dist)
    yseq = DeviceSeq(y, (n,), _lib.PMX_F32)
    prep_red = PreparedMapReduce(None, P.addf, 0.0, yseq, ctx)
    red_ms, _ = device_time(prep_red.launch, args.steps, 1, dist)
    prep_mat = PreparedMapReduce(f, P.addf, 0.0, seq, ctx, materialize=y)
    mat_ms, _ = device_time(prep_mat.launch, args.steps, 1, dist)
    ctx.check_errors()

    generic = bench_generic_skeletons(x, n, args, dist, peaks)
    kern_ms = statistics.mean(per)
    bytes_per_launch = 4 * n
    achieved = bytes_per_launch / (kern_ms * 1e-3) / 1e9

    # e2e: public accelerate entry, pinned host input, result read back
    host_x = x.to("cpu").pin_memory()
    e2e_body = lambda s: P.eval_reduce(P.addf, 0.0, P.eval_map(f, s))

    def e2e_step():
        v = P.accelerate(e2e_body, host_x)        # this rank's shard: H2D + fused kernel + D2H
        if dist.world > 1:                        # combine the per-rank partials (rank order)
            t = torch.tensor([v], dtype=torch.float64, device=dev)
            dist.all_gather(gathered, t)
            return float(prep.fold_partials(gathered).item())
        return v

    e2e_ms, e2e_wall = host_time(e2e_step, max(2, min(args.steps, 5)), 1, dist)
    e2e_steps = max(2, min(args.steps, 5))
    e2e_val = n * dist.world / (e2e_ms / e2e_steps * 1e-3)

    out = {
        "value": n * dist.world / (total_ms / args.steps * 1e-3),
        "ms_per_step": total_ms / args.steps,
        "result": result, "exact_result": exact, "result_exact_match": (result == exact) if exact else None,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": _traffic_from_profiles(),
                     "kernel": "k_map_reduce_vec<float,float,FAffineF,OAddF,false,true> (fp64 map + sum, Float semantics)",
                     "bytes_per_launch": bytes_per_launch, "kernel_ms": round(kern_ms, 5),
                     "peak_source": peaks["source"]},
        "e2e": {"value": e2e_val, "unit": "elements/s", "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 8,
                "ms_per_step": e2e_ms / e2e_steps, "path": "accelerate(reduce addf 0.0 (map f s)) with pinned host s"},
        "gpu_launches": launches,
        "combine": ("peer-memory exchange fused into the reduce kernel (pmx_map_reduce_peers)" if peers is not None
                    else ("NCCL all-gather + device fold" if dist.world > 1 else "single GPU")),
        "clocks": clk,
        "variants": {
            "map_only_8B": {"ms": map_ms / args.steps, "GB/s": 8 * n / (map_ms / args.steps * 1e-3) / 1e9,
                            "frac": 8 * n / (map_ms / args.steps * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "reduce_only_4B": {"ms": red_ms / args.steps, "GB/s": 4 * n / (red_ms / args.steps * 1e-3) / 1e9,
                               "frac": 4 * n / (red_ms / args.steps * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "map_reduce_materialised_8B": {"ms": mat_ms / args.steps,
                                           "GB/s": 8 * n / (mat_ms / args.steps * 1e-3) / 1e9,
                                           "frac": 8 * n / (mat_ms / args.steps * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "unfused_map_then_reduce_elem_per_s": n / ((map_ms + red_ms) / args.steps * 1e-3),
            "nccl_allgather_combine_ms": (nccl_ms / args.steps) if nccl_ms is not None else None,
            "generic_lambdas": generic,
        },
    }
    return out


def bench_generic_skeletons(x, n, args, dist, peaks) -> dict:
    """The skeletons on lambdas the library does not recognise (run-time
    specialised kernels, csrc/jit.cu) over the same 2^28 fp32 shard:
    map / map2 / map->reduce / loop, HBM roofline each."""
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib
    from paper_2211_00621_b200.runtime import DeviceSeq, DeviceTensor, _Root
    xs = DeviceSeq(x, (n,), _lib.PMX_F32)
    ys = DeviceSeq(torch.roll(x, 1), (n,), _lib.PMX_F32)
    yt = torch.empty_like(x)
    tx = DeviceTensor(_Root(x, 0, 0, n, _lib.PMX_F32), 0, (n,), "float")
    ty = DeviceTensor(_Root(yt, 1, 0, n, _lib.PMX_F32), 0, (n,), "float")
    f = P.lam("x", P.addf(P.mulf("x", "x"), 1.0))
    g = P.lam("a", "b", P.subf(P.mulf("a", "b"), "a"))
    sq = P.lam("x", P.mulf("x", "x"))
    body = P.lam("i", P.tensor_set(ty, ["i"], P.addf(P.mulf(2.0, P.tensor_get(tx, ["i"])), 1.0)))
    gop = P.lam("a", "b", P.addf("a", P.mulf("b", 1.0)))
    cases = [("map (lam x. x*x + 1)", lambda: P.eval_map(f, xs).materialize(), 8),
             ("map2 (lam a b. a*b - a)", lambda: P.eval_map2(g, xs, ys), 12),
             ("reduce addf 0.0 (map (lam x. x*x))", lambda: P.eval_reduce(P.addf, 0.0, P.eval_map(sq, xs)), 4),
             ("loop n (lam i. tensorSet y [i] (2*(tensorGet x [i])+1))", lambda: P.eval_loop(n, body), 8),
             ("reduce (lam a b. addf a (mulf b 1.0)) 0.0 s  [operator not recognised: ordered tree]",
              lambda: P.eval_reduce(gop, 0.0, xs), 4)]
    # seqLoop: 20 on-device steps of a 2-point stencil over 2^24 fp64 states
    # (16 B per element-step: state read + write; the neighbour read hits cache)
    ms_, steps_ = 1 << 24, 20
    s_state = DeviceSeq(torch.arange(ms_, dtype=torch.float64, device=x.device) % 97, (ms_,), _lib.PMX_F64)
    stencil = P.lam("x", "j", "t", P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 1), ms_)))))
    cases.append(("seq_loop 20 (lam x j t. 0.5*(x + get prev ((j+1) mod m))), m=2^24 fp64",
                  lambda: P.seq_loop(steps_, stencil, s_state), None))
    out = {}
    c0, l0 = _lib.jit_stats()
    for name, fn, bpe in cases:
        ms, _ = device_time(fn, args.steps, 3, dist)
        ms /= args.steps
        if bpe is None:      # seqLoop: 16 B per element-step over ms_ x steps_
            gbs = 16.0 * ms_ * steps_ / (ms * 1e-3) / 1e9
            out[name] = {"ms": round(ms, 4), "bytes_per_elem_step": 16, "GB/s": round(gbs, 1),
                         "frac": round(gbs / peaks["hbm_gbs"], 3), "elem_steps_per_s": ms_ * steps_ / (ms * 1e-3)}
            continue
        gbs = bpe * n / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 4), "bytes_per_elem": bpe, "GB/s": round(gbs, 1),
                     "frac": round(gbs / peaks["hbm_gbs"], 3), "elem_per_s": n / (ms * 1e-3)}
    c1, l1 = _lib.jit_stats()
    out["_jit"] = {"kernels_compiled": c1 - c0, "launches": l1 - l0}
    return out


def _traffic_from_profiles():
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("map_reduce")
        except Exception:
            return None
    return None


def cpu_baseline_mapreduce(seconds: float = 10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O     # CPU baseline leg only
    from paper_2211_00621_b200 import synth
    m = 1 << 26
    x = synth.mapreduce_x(m)
    th = cpu_threads()
    O.map_affine_reduce_add(x, workers=th, threads=th)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.map_affine_reduce_add(x, workers=th, threads=th)
        reps += 1
        if time.perf_counter() - t0 > seconds and reps >= 3:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": m / dt, "unit": "elements/s", "cores": th, "kind": "port",
            "sample": f"{reps} passes of the oracle (oracle/pmx_oracle.c, fp64 reference semantics, "
                      f"{th} OpenMP threads = {th} chunks) over 2^26 of the 2^28 elements"}


# ============================================================ case studies
def bench_rk4(args, dist, peaks) -> dict:
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import casestudies as CS, synth
    n, m = 10_000, 1_000
    dev = torch.device("cuda", torch.cuda.current_device())
    ps = torch.from_numpy(synth.rk4_params(n)).to(dev)
    s0 = torch.from_numpy(synth.RK4_INIT).to(dev)
    step = lambda: CS.rk4_sweep(ps, s0, m, synth.RK4_H)
    total, per = device_time(step, args.steps, args.warmup, dist)
    ms = total / args.steps
    got = step().data.view(n, 4).to("cpu").numpy()
    # FP64 work as written per param-step: 4 deriv (13 flops) + 3 axpy (8) + combine (28) = 104
    flops = 104.0 * n * m
    host_ps = ps.to("cpu").pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(lambda p, s: CS.rk4_sweep(p, s, m, synth.RK4_H), host_ps,
                                                synth.RK4_INIT), 3, 1, dist)
    return {"config": f"N={n} parameter sets x M={m} steps, fp64", "element": "parameter set",
            "value": n * dist.world / (ms * 1e-3), "ms_per_step": ms,
            "param_steps_per_s": n * m * dist.world / (ms * 1e-3),
            "e2e": {"value": n * dist.world / (e2e_ms / 3 * 1e-3), "h2d_bytes_per_step": 8 * n + 32,
                    "d2h_bytes_per_step": 32 * n},
            "roofline": {"bound": "fp64 latency (68 threads/SM at N=1e4)", "achieved_gflops": flops / (ms * 1e-3) / 1e9,
                         "note": "transcendentals (12 sin/cos per step) not counted"},
            "_result": got}


def cpu_rk4(seconds=10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    n = max(64, 16 * th)
    ps = synth.rk4_params(10_000)[:n]
    reps, t0 = 0, time.perf_counter()
    while True:
        O.rk4(ps, synth.RK4_INIT, 1000, synth.RK4_H, threads=th)
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": n / dt, "unit": "parameter sets/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {n} of the 10^4 parameter sets x 1000 steps"}


def bench_knn(args, dist, peaks) -> dict:
    import torch
    from paper_2211_00621_b200 import casestudies as CS, synth
    ntr, nq, d, k, c = 1 << 20, 1 << 16, 64, 8, 10
    dev = torch.device("cuda", torch.cuda.current_device())
    X = torch.from_numpy(synth.knn_train(ntr, d)).to(dev)
    Q = torch.from_numpy(synth.knn_query(nq, d)).to(dev)
    L = torch.from_numpy(synth.knn_labels(ntr, c)).to(dev)
    out = torch.empty(nq, dtype=torch.int32, device=dev)
    from paper_2211_00621_b200 import _lib
    ws = torch.empty(_lib.load().pmx_knn_workspace_bytes(ntr, nq, d, k), dtype=torch.uint8, device=dev)
    step = lambda: CS.knn_raw(X, L, Q, ntr, nq, d, k, c, out, None, ws)
    w, s = min(args.warmup, 2), max(1, min(args.steps, 3))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    flops = 2.0 * d * ntr * nq
    # end to end through the public entry with host arrays (H2D of train,
    # labels, queries + kernels + D2H of the labels)
    import paper_2211_00621_b200 as P
    hX, hQ, hL = X.cpu().pin_memory(), Q.cpu().pin_memory(), L.cpu().pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(lambda a, b, q: P.knn_classify(a, b, q, k, c), hX, hL, hQ),
                          2, 1, dist)
    e2e = {"value": nq * dist.world / (e2e_ms / 2 * 1e-3), "unit": "queries/s",
           "h2d_bytes_per_step": hX.numel() * 4 + hQ.numel() * 4 + hL.numel() * 4, "d2h_bytes_per_step": nq * 4}
    return {"config": "2^20 train x 2^16 queries, d=64, k=8, 10 classes, fp32", "element": "query",
            "value": nq * dist.world / (ms * 1e-3), "ms_per_step": ms, "steps": s, "warmup": w, "e2e": e2e,
            "pair_dims_per_s": float(ntr) * nq * d * dist.world / (ms * 1e-3),
            "roofline": {"bound": "TMEM read (one fp32 distance per candidate leaves TMEM)",
                         "achieved_tflops": flops / (ms * 1e-3) / 1e12,
                         "peak_tflops": peaks["bf16_tflops"],
                         "frac": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                         "tmem_read_bytes": 4.0 * ntr * nq,
                         "tmem_read_B_per_clk_per_sm": 4.0 * ntr * nq / (ms * 1e-3) / 148 / 1.965e9,
                         "note": "tcgen05 bf16 UMMA (exact for the integer data) with ||x||^2 folded into an "
                                 "augmentation k-step; TMEM->RF at ~64 B/clk/SM (B300_MICROARCH) bounds it"},
            "_labels": out.to("cpu").numpy()}


def cpu_knn(seconds=10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    X = synth.knn_train(1 << 20, 64)
    L = synth.knn_labels(1 << 20, 10)
    nq = max(8, th)
    Q = synth.knn_query(nq, 64)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.knn(X, L, Q, 8, 10, threads=th)
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": nq / dt, "unit": "queries/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {nq} of the 2^16 queries against all 2^20 train points"}


def bench_hmm(args, dist, peaks) -> dict:
    import torch
    from paper_2211_00621_b200 import _lib, casestudies as CS, synth
    S, K, nsig, T = 1024, 8, 4096, 10_000
    dev = torch.device("cuda", torch.cuda.current_device())
    A, E, pi = synth.hmm_model(S, K)
    import numpy as np
    Ad = torch.from_numpy(A.astype(np.float32)).to(dev)
    lE = torch.from_numpy(np.log(E).astype(np.float32)).to(dev)
    lpi = torch.from_numpy(np.log(pi).astype(np.float32)).to(dev)
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).to(dev)
    out = torch.empty(nsig, dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.load().pmx_hmm_forward_workspace_bytes(S, nsig), dtype=torch.uint8, device=dev)
    step = lambda: CS.hmm_forward_raw(lpi, Ad, lE, obs, S, K, nsig, T, out, ws)
    w, s = min(args.warmup, 1), max(1, min(args.steps, 2))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    # end to end through the public entry with host arrays (probabilities and
    # observations H2D, logs on the device, kernel, log-likelihoods D2H)
    import paper_2211_00621_b200 as P
    hobs = obs.cpu().pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(P.hmm_forward, A, E, pi, hobs), 1, 1, dist)
    e2e = {"value": nsig * dist.world / (e2e_ms * 1e-3), "unit": "signals/s",
           "h2d_bytes_per_step": hobs.numel() * 4 + 8 * (A.size + E.size + pi.size), "d2h_bytes_per_step": 8 * nsig}
    flops = 2.0 * S * S * (T - 1) * nsig
    # 4-CTA kernel (hmm_quad.cu), per SM per step: its 256 rows of A^T written by
    # TMA and read by the pair UMMAs (fp16), its 64-signal B half re-read once per
    # M block (2 x 1024 x 64 fp16), and the u_t rows written locally / received
    # (1024 states x 64 signals fp16) plus the staging rows (2 x 16 KiB)
    rows = S // 4
    smem_step = 2 * rows * S * 2 + 2 * S * 64 * 2 + S * 64 * 2 + 2 * 16384
    smem_peak = pipe_peaks().get("per_sm_per_clk_at_attr_clock", {}).get("smem_load_B", 128.0)
    return {"config": "4096 signals x 10^4 steps x 1024 states, K=8, fp16 operands / fp32 accumulate + fp64 log-scale",
            "element": "signal", "value": nsig * dist.world / (ms * 1e-3), "ms_per_step": ms,
            "steps": s, "warmup": w, "e2e": e2e,
            "trellis_cells_per_s": float(S) * S * (T - 1) * nsig * dist.world / (ms * 1e-3),
            "roofline": {"bound": "tensor pipe / per-step synchronisation (u_t exchanged between 4 SMs every step)",
                         "achieved_tflops": flops / (ms * 1e-3) / 1e12,
                         "peak_tflops": peaks["bf16_tflops"],
                         "peak_source": "f16 dense = measured bf16 dense (MEASURED_PEAKS.json)",
                         "frac": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                         "smem_bytes_per_sm_per_step": smem_step,
                         "smem_B_per_clk_per_sm": smem_step * (T - 1) / (ms * 1e-3) / 1.965e9,
                         "smem_frac": smem_step * (T - 1) / (ms * 1e-3) / 1.965e9 / smem_peak,
                         "umma_probe_tflops": {"M128_N64": 1463.4, "M128_N128": 2205.1,
                                               "source": "tools/umma_rate.cu (profiles/umma_rate.json)"},
                         "note": "tcgen05 kind::f16 cta_group::2 (M = 256 across a CTA pair, N = 128 signals split "
                                 "64/64 between the pair's B buffers), 2^10-scaled fp16 operands, fp32 TMEM "
                                 "accumulation; clusters of 4 (two pairs split the states); u_t rows exchanged by "
                                 "DSMEM bulk copies, consumed by the next step's UMMAs per (source CTA, M block) as "
                                 "they land (TMEM D double-buffered). CTA-pair kernel with single-SM UMMAs "
                                 "(PMX_HMM_TC=pair): 13.2 us/step"},
            "_ll": out.to("cpu").numpy()}


def cpu_hmm(seconds=10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    A, E, pi = synth.hmm_model(1024, 8)
    T = 20
    obs = synth.hmm_obs(max(2, th), T, 8)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.hmm_forward(A, E, pi, obs, threads=th)
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    sig_steps = obs.shape[0] * (T - 1) / dt
    return {"value": sig_steps / (10_000 - 1), "unit": "signals/s (T=10^4 equivalent)", "cores": th, "kind": "port",
            "sample": f"{reps}x {obs.shape[0]} signals x {T} steps at S=1024 (log-space oracle), scaled to T=10^4"}


def bench_viterbi(args, dist, peaks) -> dict:
    """Viterbi decoding (programs/viterbi.pmx) at scale: SURVEY §8(f) rank 1.
    Not a BASELINE config: the HMM model of the forward config (S=1024, K=8),
    1184 signals (8 per SM) x T=1000, fp64 like the reference."""
    import numpy as np
    import torch
    from paper_2211_00621_b200 import _lib, synth
    S, K, nsig, T = 1024, 8, 148 * 8, 1000
    dev = torch.device("cuda", torch.cuda.current_device())
    A, E, pi = synth.hmm_model(S, K)
    lA = torch.from_numpy(np.log(A)).to(dev)
    lE = torch.from_numpy(np.log(E)).to(dev)
    lpi = torch.from_numpy(np.log(pi)).to(dev)
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).to(dev)
    path = torch.empty(nsig * T, dtype=torch.int32, device=dev)
    logp = torch.empty(nsig, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pmx_viterbi_workspace_bytes(S, nsig, T), dtype=torch.uint8, device=dev)

    def step():
        _lib.check(lib.pmx_viterbi_f64(lpi.data_ptr(), lA.data_ptr(), lE.data_ptr(), S, K, obs.data_ptr(), nsig,
                                       T, path.data_ptr(), logp.data_ptr(), ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream().cuda_stream), "viterbi")
    w, s = min(args.warmup, 1), max(1, min(args.steps, 2))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    cells = float(S) * S * (T - 1) * nsig
    pp = pipe_peaks()
    fp64_lanes = pp.get("fp64_add_ops_per_s", 64.0 * 148 * 1.965e9)   # FP64 pipe ops/s
    return {"config": f"S={S}, K={K}, {nsig} signals x T={T}, fp64 (viterbi.pmx semantics)", "element": "signal",
            "value": nsig * dist.world / (ms * 1e-3), "ms_per_step": ms, "steps": s, "warmup": w,
            "cells_per_s": cells / (ms * 1e-3),
            "roofline": {"bound": "dense-equivalent max-plus cells (2 FP64 ops each); the default kernel "
                                  "prunes each column's scan (sorted logA, exact bound) and visits ~7-15% of them",
                         "achieved_fp64_ops_per_s": 2 * cells / (ms * 1e-3), "peak_fp64_ops_per_s": fp64_lanes,
                         "frac": 2 * cells / (ms * 1e-3) / fp64_lanes,
                         "issue_frac": 5 * cells / (ms * 1e-3) / (128.0 * 148 * 1.965e9),
                         "peak_source": ("measured (profiles/pipe_peaks.json, tools/peaks.cu)" if pp else
                                         "64 FP64 lanes/clk/SM x 148 SMs x 1.965 GHz") +
                                        "; issue: 4 x 32 thread-instr/clk/SM"},
            "_path": path}


def cpu_viterbi(seconds=10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    A, E, pi = synth.hmm_model(1024, 8)
    T = 20
    obs = synth.hmm_obs(max(2, th), T, 8)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.viterbi(A, E, pi, obs, threads=th)
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": obs.shape[0] * (T - 1) / dt / (1000 - 1), "unit": "signals/s (T=1000 equivalent)",
            "cores": th, "kind": "port", "sample": f"{reps}x {obs.shape[0]} signals x {T} steps at S=1024"}


def bench_nn(args, dist, peaks) -> dict:
    """Softmax-regression loss + gradients (programs/nn.pmx) at scale: SURVEY
    §8(f) rank 3.  2^20 points, 64 inputs, 16 classes, fp64 (the reference's
    Float); x is the only HBM stream (512 MiB)."""
    import numpy as np
    import torch
    from paper_2211_00621_b200 import _lib
    npts, nin, nout = 1 << 20, 64, 16
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn(npts * nin, dtype=torch.float64, device=dev, generator=g) * 0.5
    y = torch.randint(0, nout, (npts,), dtype=torch.int32, device=dev, generator=g)
    w = torch.randn(nin * nout, dtype=torch.float64, device=dev, generator=g) * 0.3
    b = torch.randn(nout, dtype=torch.float64, device=dev, generator=g) * 0.1
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    dw = torch.empty(nin * nout, dtype=torch.float64, device=dev)
    db = torch.empty(nout, dtype=torch.float64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    lib = _lib.load()
    ws = torch.zeros(lib.pmx_nn_workspace_bytes(npts, nin, nout), dtype=torch.uint8, device=dev)

    def step():
        _lib.check(lib.pmx_nn_softmax_grad_f64(x.data_ptr(), y.data_ptr(), w.data_ptr(), b.data_ptr(), npts, nin,
                                               nout, loss.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(),
                                               ws.numel(), err.data_ptr(), torch.cuda.current_stream().cuda_stream),
                   "nn")
    total, per = device_time(step, args.steps, args.warmup, dist)
    ms = total / args.steps
    bytes_ = 8.0 * nin * npts + 4.0 * npts
    flops = npts * (2.0 * nin * nout * 2)            # z (mul+add) and dw (mul+add), fp64
    pipe_ops = npts * (3.0 * nin * nout)             # z: DMUL + DADD; dw: one DFMA
    pp = pipe_peaks()
    fp64_ops_peak = pp.get("fp64_add_ops_per_s", 64.0 * 148 * 1.965e9)
    return {"config": f"{npts} points x {nin} inputs x {nout} classes, fp64 (nn.pmx semantics)", "element": "point",
            "value": npts * dist.world / (ms * 1e-3), "ms_per_step": ms,
            "roofline": {"bound": "HBM (x stream) / FP64 pipe", "achieved_GBps": bytes_ / (ms * 1e-3) / 1e9,
                         "hbm_frac": bytes_ / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "achieved_fp64_tflops": flops / (ms * 1e-3) / 1e12,
                         "fp64_pipe_ops_per_s": pipe_ops / (ms * 1e-3),
                         "fp64_pipe_frac": pipe_ops / (ms * 1e-3) / fp64_ops_peak,
                         "peak_source": "HBM: MEASURED_PEAKS.json; FP64 pipe: " +
                                        ("measured (profiles/pipe_peaks.json)" if pp else "64 lanes/clk/SM nominal"),
                         "note": "z keeps the reference's separately rounded mul + add (2 pipe ops per MAC); "
                                 "dw sums use DFMA (1 pipe op)"},
            "_loss": float(loss.item())}


def pipe_peaks() -> dict:
    """FP64 / FP32 / MUFU / shared-memory rates measured on a B200 by
    tools/peaks.cu (profiles/pipe_peaks.json); {} when absent."""
    f = ROOT / "profiles" / "pipe_peaks.json"
    try:
        return json.loads(f.read_text())
    except (OSError, ValueError):
        return {}


def cpu_nn(seconds=10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np
    import oracle as O
    n, nin, nout = 1 << 16, 64, 16
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, nin))
    y = rng.integers(0, nout, n).astype(np.int32)
    w = rng.standard_normal((nin, nout))
    b = rng.standard_normal(nout)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.nn(x, y, w, b, workers=1)
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": n / dt, "unit": "points/s", "cores": 1, "kind": "port",
            "sample": f"{reps}x 2^16 of the 2^20 points (oracle_nn is single-threaded)"}


def bench_kmer(args, dist, peaks) -> dict:
    import numpy as np
    import torch
    from paper_2211_00621_b200 import _lib, casestudies as CS, synth
    kmer, K, T = 8, 8, 6000
    nsig = 8192 // 8       # this GPU's share of 8k signals over 8 GPUs
    dev = torch.device("cuda", torch.cuda.current_device())
    lE = torch.from_numpy(np.log(synth.kmer_emission(kmer, K)).astype(np.float32)).to(dev)
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).to(dev)
    out = torch.empty(nsig, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pmx_hmm_kmer_workspace_bytes(kmer, nsig), dtype=torch.uint8, device=dev)

    def step():
        rc = lib.pmx_hmm_kmer_forward_f32(kmer, 0.5, 0.125, lE.data_ptr(), K, obs.data_ptr(), nsig, T,
                                          out.data_ptr(), ws.data_ptr(), ws.numel(),
                                          torch.cuda.current_stream().cuda_stream)
        _lib.check(rc, "kmer")
    w, s = min(args.warmup, 1), max(1, min(args.steps, 2))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    S = 1 << (2 * kmer)
    # per signal-step: alpha stay reads + step-predecessor reads + writes + emission row, 4 B each
    bytes_ = 4.0 * 4 * S * (T - 1) * nsig
    return {"config": "S=65536 (k=8) de Bruijn, 1024 signals per GPU (8192 over 8), T=6000, fp32",
            "element": "signal", "value": nsig * dist.world / (ms * 1e-3), "ms_per_step": ms,
            "steps": s, "warmup": w,
            "trellis_cells_per_s": 5.0 * S * (T - 1) * nsig * dist.world / (ms * 1e-3),
            "roofline": {"bound": "L2 (alpha slices L2-resident, streamed every step)",
                         "achieved_l2_GBps": bytes_ / (ms * 1e-3) / 1e9,
                         "vs_hbm_peak": bytes_ / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "bytes_per_signal_step": 16 * S,
                         "l2_probe_GBps": {k: v / 1e9 for k, v in pipe_peaks().items()
                                           if k.startswith("l2_read_bytes_per_s")},
                         "note": "algorithmic L2 bytes (stay + step-predecessor reads, emission row, write: "
                                 "16 B per state-step); the alpha working set (148 x 512 KiB) stays L2-resident "
                                 "(DRAM traffic ~0 in ncu). The L2 probe (tools/peaks.cu, a simple streaming "
                                 "kernel) is a lower bound on the L2 peak: this kernel exceeds it"},
            "_ll": out.to("cpu").numpy()}


def cpu_kmer(seconds=10.0) -> dict:
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    E = synth.kmer_emission(8, 8)
    T = 30
    obs = synth.hmm_obs(max(2, th), T, 8)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.kmer_forward(8, 0.5, 0.125, E, obs, threads=th)
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": obs.shape[0] * (T - 1) / dt / (6000 - 1), "unit": "signals/s (T=6000 equivalent)",
            "cores": th, "kind": "port", "sample": f"{reps}x {obs.shape[0]} signals x {T} steps at S=65536"}


# ================================================================= main
def run_ours(args):
    import torch
    dist = Dist()
    torch.cuda.set_device(dist.local % max(1, torch.cuda.device_count()))
    dist.init("nccl")
    import paper_2211_00621_b200 as P
    P.load_library()
    peaks = _peaks()
    res = bench_mapreduce(args, dist, peaks)
    cpu = cpu_baseline_mapreduce(args.cpu_seconds) if (dist.rank == 0 and dist.world == 1 and not args.no_cpu) else None
    case = {}
    if not args.no_case_studies:
        for name, fn, cfn in (("rk4", bench_rk4, cpu_rk4), ("knn", bench_knn, cpu_knn),
                              ("hmm_forward", bench_hmm, cpu_hmm), ("hmm_kmer", bench_kmer, cpu_kmer),
                              ("viterbi", bench_viterbi, cpu_viterbi), ("nn", bench_nn, cpu_nn)):
            if args.case and name not in args.case:
                continue
            try:
                r = fn(args, dist, peaks)
                r = {k: v for k, v in r.items() if not k.startswith("_")}
                if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
                    r["cpu_baseline"] = cfn(args.cpu_seconds / 2)
                    r["speedup_vs_cpu"] = r["value"] / r["cpu_baseline"]["value"]
                case[name] = r
            except Exception as exc:    # report, do not hide
                case[name] = {"error": f"{type(exc).__name__}: {exc}"}
    if dist.rank != 0:
        return
    line = {
        "metric": METRIC, "value": res["value"], "unit": "elements/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (integer-formula inputs, SURVEY §8(d))",
        "config": {"workload": "map/reduce skeleton microbench: reduce addf 0.0 (map (lam x. 2x+1) s), "
                               "2^28 fp32 elements per GPU (BASELINE configs[1]), fused map->reduce",
                   "n_per_gpu": N_PER_GPU, "n_total": N_PER_GPU * dist.world,
                   "parallelism": f"data-parallel x{dist.world} (contiguous shards + NCCL all-gather of partials)",
                   "l2": "inputs (1 GiB/GPU) larger than L2 (126 MB); no flush needed"},
        "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"], "gpu_launches": res["gpu_launches"],
        "clocks": res["clocks"], "result": {"sum": res["result"], "exact": res["exact_result"],
                                            "bit_exact": res["result_exact_match"]},
        "variants": res["variants"], "case_studies": case,
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference arm: the CPU restatement of the reference's path (the
    oracle port, oracle/pmx_oracle.c) on this box's host cores, same metric and
    workload; rank 0 only."""
    dist = Dist()
    if dist.rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np
    import oracle as O
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    n = N_PER_GPU
    x = synth.mapreduce_x(n)
    per = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.map_affine_reduce_add(x, workers=th, threads=th)
        if i >= args.warmup:
            per.append(time.perf_counter() - t0)
    ms = 1e3 * sum(per) / len(per)
    val = n / (ms * 1e-3)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "elements/s", "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (integer-formula inputs, SURVEY §8(d))",
            "config": {"workload": "map/reduce skeleton microbench: reduce addf 0.0 (map (lam x. 2x+1) s), "
                                   "2^28 elements (BASELINE configs[1])", "n_per_gpu": n, "n_total": n},
            "cpu_baseline": {"value": val, "unit": "elements/s", "cores": th, "kind": "port",
                             "sample": "full 2^28-element workload per step; oracle/pmx_oracle.c "
                                       "oracle_map_affine_reduce_add (fp64 Float semantics, _chunks partition)"},
            "e2e": {"value": val, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-case-studies", action="store_true")
    ap.add_argument("--case", action="append", default=[])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines (quick experiments)")
    ap.add_argument("--nccl-combine", action="store_true",
                    help="N>1: combine reduce partials with NCCL all-gather instead of the fused peer kernel")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

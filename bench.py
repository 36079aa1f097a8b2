"""Benchmark of the accelerated-expression hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--case NAME ...] [--no-case-studies] [--no-cpu] [--no-parity]

`--gpus N` with no torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU; PMX_DIST_BACKEND=gloo lets
N ranks share one GPU as a functional check).

Headline workload (BASELINE.json configs[1]): the map/reduce skeleton
microbench — `reduce addf 0.0 (map (lam x. addf (mulf 2.0 x) 1.0) s)` over
2^28 fp32 elements per GPU (weak scaling: rank r owns elements
[r*2^28, (r+1)*2^28) of an N*2^28-element sequence, the _chunks partition of
pmx/interp.py:273-276; the per-rank partials meet in the reduce kernel itself
over NVLink peer memory).  One step = one evaluation of that expression.
Inputs (1 GiB per GPU) are larger than L2 (126 MB), so no flush is needed.

`value` is device-resident throughput (elements/s, all ranks), `e2e` the same
program through the public `accelerate` entry with pinned HOST input (H2D of
the input + kernel + D2H of the result inside the timed region).  The case
studies (RK4, k-NN, HMM forward, k-mer HMM, plus Viterbi and NN gradients of
SURVEY §8(f)) are reported under `case_studies`, each with its own roofline,
end-to-end number, CPU-port baseline and a `parity` block that checks the
timed outputs against the CPU oracle (sampled at full size).  The reference
arm (`--impl reference`) prints the same line for the CPU port of the
reference's path, with the same `config` and `case_studies` configs.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import socket
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


def pipe_peaks() -> dict:
    """FP64 / FP32 / MUFU / shared-memory / L2 rates measured on a B200 by
    tools/peaks.cu (profiles/pipe_peaks.json); {} when absent."""
    f = ROOT / "profiles" / "pipe_peaks.json"
    try:
        return json.loads(f.read_text())
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------- configs
# One source for the `config` dicts of both arms (the driver compares them).
def headline_config(world: int) -> dict:
    return {"workload": "map/reduce skeleton microbench: reduce addf 0.0 (map (lam x. 2x+1) s), "
                        "2^28 fp32 elements per GPU (BASELINE configs[1]), fused map->reduce",
            "n_per_gpu": N_PER_GPU, "n_total": N_PER_GPU * world,
            "arithmetic": "fp64 (the reference's Float) over fp32 storage",
            "parallelism": f"data-parallel x{world}: contiguous _chunks shards, partials combined in rank order",
            "l2": "inputs (1 GiB/GPU) larger than L2 (126 MB); no flush needed"}


def case_configs(world: int) -> dict:
    return {
        "rk4": {"workload": f"RK4 sweep, {10_000 * world} parameter sets (10^4 per GPU) x 10^3 steps, fp64, "
                            "p_k = 0.5 + k/N (BASELINE configs[0])", "element": "parameter set",
                "unit": "parameter sets/s"},
        "knn": {"workload": f"k-NN: 2^20 train x {65536 * world} queries (2^16 per GPU), d=64, k=8, 10 classes, "
                            "fp32 integer-valued coordinates (BASELINE configs[2])", "element": "query",
                "unit": "queries/s"},
        "hmm_forward": {"workload": f"HMM forward: {4096 * world} signals (4096 per GPU) x T=10^4 x S=1024, K=8, "
                                    "log-likelihood in fp64 (BASELINE configs[3])", "element": "signal",
                        "unit": "signals/s"},
        "hmm_kmer": {"workload": f"HMM forward, k-mer model S=65536 (k=8), {1024 * world} signals (8192 over 8 "
                                 "GPUs: 1024 per GPU) x T=6000 (BASELINE configs[4])", "element": "signal",
                     "unit": "signals/s"},
        "viterbi": {"workload": f"Viterbi (programs/viterbi.pmx), S=1024, K=8, {1184 * world} signals (1184 per "
                                "GPU) x T=1000, fp64 (SURVEY §8(f) rank 1)", "element": "signal",
                    "unit": "signals/s"},
        "nn": {"workload": f"softmax-regression loss + gradients (programs/nn.pmx), {(1 << 20) * world} points "
                           "(2^20 per GPU) x 64 inputs x 16 classes, fp64 (SURVEY §8(f) rank 3)",
               "element": "point", "unit": "points/s"},
    }


# ------------------------------------------------------------- distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None

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
        import torch
        if self.backend == "nccl":
            self.pg.all_gather_into_tensor(out, t)
            return
        parts = [torch.empty(t.shape, dtype=t.dtype) for _ in range(self.world)]
        self.pg.all_gather(parts, t.cpu())
        out.copy_(torch.cat(parts).to(out.device))

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def shard(self, n_global: int) -> tuple[int, int]:
        from paper_2211_00621_b200.shard import chunk
        return chunk(n_global, self.world, self.rank)


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
def device_time(step, steps: int, warmup: int, dist: Dist):
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


def pcie_h2d_gbs(nbytes: int = 1 << 30) -> float:
    """Pinned host -> device copy bandwidth (GB/s, best of 6) at the headline's
    1 GiB: the bound of any end-to-end number whose inputs start in host
    memory (tools/h2d_probe.py: one stream or the bytes split over 2 / 4
    streams copy at the same 55.5 GB/s, i.e. the link, not a copy engine)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O     # the checker / CPU baseline only
    return O


def _e2e(value_unit: str, n_elems: int, ms: float, h2d: int, d2h: int, pcie: float | None, path: str) -> dict:
    out = {"value": n_elems / (ms * 1e-3), "unit": value_unit, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "path": path}
    if pcie:
        bound_ms = (h2d + d2h) / (pcie * 1e9) * 1e3
        out["pcie"] = {"h2d_GBps_measured": round(pcie, 1), "copy_ms_at_that_rate": round(bound_ms, 3),
                       "frac_of_step_in_copies": round(bound_ms / ms, 3)}
    return out


# ============================================================ map/reduce
def bench_mapreduce(args, dist: Dist, peaks: dict, pcie: float | None) -> dict:
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
    # N > 1: the shard partials meet inside the reduce kernel over NVLink peer
    # memory (one launch per step, no collective); acc is rank 0's (shard.py).
    # The NCCL all-gather + fold is timed beside it as a variant.
    from paper_2211_00621_b200.shard import PeerMailboxes, ShardedMapReduce
    peers = PeerMailboxes() if (dist.world > 1 and not args.nccl_combine) else None
    smr = ShardedMapReduce(f, P.addf, 0.0, seq, n * dist.world, ctx=ctx, peers=peers)
    step = smr.launch

    launches0 = ctx.launches
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    total_ms, per = device_time(step, args.steps, args.warmup, dist)
    clk = clocks.stop()
    launches = (ctx.launches - launches0) // (args.steps + args.warmup) * args.steps
    result = float(step().item())
    nccl_ms = None
    if dist.world > 1:
        nccl = ShardedMapReduce(f, P.addf, 0.0, seq, n * dist.world, ctx=ctx, peers=None)
        nccl_ms, _ = device_time(nccl.launch, args.steps, 1, dist)
    ctx.check_errors()
    exact = synth.mapreduce_exact_sum(n * dist.world)

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
    map_ok = bool(torch.equal(y, x * 2 + 1)) if not args.no_parity else None

    generic = bench_generic_skeletons(x, n, args, dist, peaks)
    kern_ms = statistics.mean(per)
    bytes_per_launch = 4 * n
    achieved = bytes_per_launch / (kern_ms * 1e-3) / 1e9

    # e2e: public accelerate entry, pinned host input (this rank's shard), result read back
    host_x = x.to("cpu").pin_memory()
    e2e_body = lambda s: P.eval_reduce(P.addf, 0.0, P.eval_map(f, s))
    gathered = torch.empty(dist.world, dtype=torch.float64, device=dev)

    def e2e_step():
        v = P.accelerate(e2e_body, host_x)        # H2D + fused kernel + D2H
        if dist.world > 1:                        # per-rank partials, folded in rank order
            dist.all_gather(gathered, torch.tensor([v], dtype=torch.float64, device=dev))
            return float(gathered.sum().item())
        return v

    e2e_steps = max(2, min(args.steps, 5))
    e2e_ms, _ = host_time(e2e_step, e2e_steps, 1, dist)
    e2e = _e2e("elements/s", n * dist.world, e2e_ms / e2e_steps, 4 * n, 8, pcie,
               "accelerate(reduce addf 0.0 (map f s)) with pinned host s")
    if pcie:
        e2e["roofline"] = {"bound": "pcie (host -> device copy of the 4-byte elements)",
                           "achieved": round(4 * n / (e2e_ms / e2e_steps * 1e-3) / 1e9, 1),
                           "peak": round(pcie, 1), "unit": "GB/s",
                           "frac": round(4 * n / (e2e_ms / e2e_steps * 1e-3) / 1e9 / pcie, 4)}

    return {
        "value": n * dist.world / (total_ms / args.steps * 1e-3),
        "ms_per_step": total_ms / args.steps,
        "result": result, "exact_result": exact,
        "parity": {"sum_bit_exact": result == exact, "exact_sum": exact,
                   "map_materialised_bit_exact": map_ok,
                   "how": "fp64 reference sum is exact for this input (SURVEY §8(d)); the map output equals 2x+1 "
                          "element for element"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": _traffic_from_profiles(),
                     "kernel": "k_map_reduce_vec<float,float,FAffineF,OAddF,false,true> (fp64 map + sum, Float semantics)",
                     "bytes_per_launch": bytes_per_launch, "kernel_ms": round(kern_ms, 5),
                     "peak_source": peaks["source"]},
        "e2e": e2e,
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


def _traffic_from_profiles(key: str = "map_reduce"):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(key)
        except Exception:
            return None
    return None


# ============================================================ case studies
def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def bench_rk4(args, dist, peaks, pcie) -> dict:
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import casestudies as CS, synth
    n_gpu, m = 10_000, 1_000
    N = n_gpu * dist.world
    lo, hi = dist.shard(N)
    n = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device())
    host_ps = synth.rk4_params(n, first=lo, total=N)
    ps = torch.from_numpy(host_ps).to(dev)
    s0 = torch.from_numpy(synth.RK4_INIT).to(dev)
    step = lambda: CS.rk4_sweep(ps, s0, m, synth.RK4_H)
    total, per = device_time(step, args.steps, args.warmup, dist)
    ms = total / args.steps
    got = step().data.view(n, 4).to("cpu").numpy()
    pinned = torch.from_numpy(host_ps).pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(lambda p, s: CS.rk4_sweep(p, s, m, synth.RK4_H), pinned,
                                                synth.RK4_INIT), 3, 1, dist)
    # Algorithmic FP64 work per parameter-step: the program as written (~104
    # add/mul and a full sin/cos per stage, 12 per step) costs 272 FP64 pipe
    # instructions per param-step (ncu thread-level DADD + DMUL + DFMA of k_rk4
    # with a full fdlibm-class sin/cos per stage, profiles/rk4_fp64.json). The
    # default kernel does less trig work (angle addition), so this
    # fixed figure over its time is the algorithmic rate, not its own count
    pp = pipe_peaks()
    prof = _rk4_profile()
    fp64_peak = pp.get("fp64_add_ops_per_s", 63.0 * 148 * 1.965e9)
    roof = {"bound": "fp64 pipe, latency-limited: N = 10^4 threads = 68 per SM (2 warps per SM sub-partition); "
                     "work = the as-written evaluation's 272 FP64 pipe instructions per param-step",
            "unit": "fp64 pipe instr/s", "peak": fp64_peak,
            "peak_source": "tools/peaks.cu (profiles/pipe_peaks.json): 63 DADD/DFMA per clk per SM"}
    if prof:
        achieved = prof["fp64_inst_per_param_step"] * n * m / (ms * 1e-3)
        roof.update({"achieved": achieved, "frac": round(achieved / fp64_peak, 4),
                     "fp64_inst_per_param_step": prof["fp64_inst_per_param_step"],
                     "ncu": prof})
    res = {"value": N / (ms * 1e-3), "ms_per_step": ms, "param_steps_per_s": N * m / (ms * 1e-3),
           "e2e": _e2e("parameter sets/s", N, e2e_ms / 3, 8 * n, 32 * n, pcie,
                       "accelerate(rk4_sweep) with pinned host parameters"),
           "roofline": roof, "kernels_per_step": 1}
    if not args.no_parity:
        O = _oracle()
        want = O.rk4(host_ps, synth.RK4_INIT, m, synth.RK4_H)
        import numpy as np
        rel = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))
        res["parity"] = {"checked": f"all {n} parameter sets x 4 components of this rank", "max_rel": rel,
                         "tolerance": 1e-9, "pass": bool(rel <= 1e-9)}
    return res


def _profile(name: str) -> dict:
    """A kernel summary distilled from this round's ncu captures (profiles/)."""
    try:
        return json.loads((ROOT / "profiles" / name).read_text())
    except (OSError, ValueError):
        return {}


def _rk4_profile() -> dict | None:
    return _profile("rk4_fp64.json") or None


def bench_knn(args, dist, peaks, pcie) -> dict:
    import numpy as np
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib, casestudies as CS, synth
    ntr, nq_gpu, d, k, c = 1 << 20, 1 << 16, 64, 8, 10
    NQ = nq_gpu * dist.world
    lo, hi = dist.shard(NQ)
    nq = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device())
    hX, hL, hQ = synth.knn_train(ntr, d), synth.knn_labels(ntr, c), synth.knn_query(nq, d, first=lo)
    X, L, Q = (torch.from_numpy(a).to(dev) for a in (hX, hL, hQ))
    out = torch.empty(nq, dtype=torch.int32, device=dev)
    idx = torch.empty(nq * k, dtype=torch.int32, device=dev)
    ws = torch.empty(_lib.load().pmx_knn_workspace_bytes(ntr, nq, d, k), dtype=torch.uint8, device=dev)
    step = lambda: CS.knn_raw(X, L, Q, ntr, nq, d, k, c, out, idx, ws)
    w, s = min(args.warmup, 2), max(1, min(args.steps, 3))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    flops = 2.0 * d * ntr * nq
    pX, pL, pQ = (torch.from_numpy(a).pin_memory() for a in (hX, hL, hQ))
    e2e_ms, _ = host_time(lambda: P.accelerate(lambda a, b, q: P.knn_classify(a, b, q, k, c), pX, pL, pQ),
                          2, 1, dist)
    achieved = flops / (ms * 1e-3) / 1e12
    res = {"value": NQ / (ms * 1e-3), "ms_per_step": ms, "steps": s, "warmup": w,
           "pair_dims_per_s": float(ntr) * NQ * d / (ms * 1e-3),
           "e2e": _e2e("queries/s", NQ, e2e_ms / 2, pX.numel() * 4 + pQ.numel() * 4 + pL.numel() * 4, nq * 4,
                       pcie, "accelerate(knn_classify) with pinned host train / labels / queries"),
           "roofline": {"bound": "tensor (int8)", "unit": "TOP/s", "achieved": achieved,
                        "peak": 2.0 * peaks["bf16_tflops"], "frac": achieved / (2.0 * peaks["bf16_tflops"]),
                        "peak_source": "int8 dense = 2 x the measured bf16 dense peak (MEASURED_PEAKS.json, burst; "
                                       "B200_PROFILING.md: int8/fp8 dense = 2 x bf16); the UMMA issue probe "
                                       "reaches 4.53 POP/s kind::i8 (profiles/umma_rate.json)",
                        "frac_vs_bf16_peak": achieved / peaks["bf16_tflops"],
                        "algorithmic_flops_per_query": 2 * d * ntr,
                        "tmem_read_bytes": 4.0 * ntr * nq,
                        "tmem_read_probe_B_per_clk_per_SM": 451,
                        "note": "tcgen05 kind::i8 UMMA on int8 operands (the integer data are exact in int8; bf16 "
                                "form for data that are not) with exact int32 accumulation of ||x||^2 - 2q.x + "
                                "||q||^2 (norms folded into an augmentation k-step); candidates leave TMEM as "
                                "packed u16 distances (tcgen05.ld .pack::16b). Not TMEM-bound (451 B/clk/SM with "
                                "16 warps); shared-memory operand traffic and the two-buffer epilogue coupling "
                                "bound it (DESIGN.md section 3)"},
           "kernels_per_step": 3}
    if not args.no_parity:
        O = _oracle()
        sel = synth.parity_sample(nq, 256)
        wl, wi = O.knn(hX, hL, hQ[sel], k, c)
        gl = out.to("cpu").numpy()[sel]
        gi = idx.to("cpu").numpy().reshape(nq, k)[sel]
        res["parity"] = {"checked": f"{len(sel)} sampled queries of this rank vs the oracle (labels and "
                                    "neighbour indices)",
                         "labels_bit_exact": bool(np.array_equal(gl, wl)),
                         "indices_bit_exact": bool(np.array_equal(gi, wi)),
                         "pass": bool(np.array_equal(gl, wl) and np.array_equal(gi, wi))}
    return res


def bench_hmm(args, dist, peaks, pcie) -> dict:
    import numpy as np
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib, casestudies as CS, synth
    S, K, ns_gpu, T = 1024, 8, 4096, 10_000
    NS = ns_gpu * dist.world
    lo, hi = dist.shard(NS)
    nsig = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device())
    A, E, pi = synth.hmm_model(S, K)
    Ad = torch.from_numpy(A.astype(np.float32)).to(dev)
    lE = torch.from_numpy(np.log(E).astype(np.float32)).to(dev)
    lpi = torch.from_numpy(np.log(pi).astype(np.float32)).to(dev)
    hobs = synth.hmm_obs(nsig, T, K, first=lo)
    obs = torch.from_numpy(hobs).to(dev)
    out = torch.empty(nsig, dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.load().pmx_hmm_forward_workspace_bytes(S, nsig), dtype=torch.uint8, device=dev)
    step = lambda: CS.hmm_forward_raw(lpi, Ad, lE, obs, S, K, nsig, T, out, ws)
    w, s = min(args.warmup, 1), max(1, min(args.steps, 2))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    rerun = CS.hmm_forward_rerun_count(S, nsig, ws)
    pobs = torch.from_numpy(hobs).pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(P.hmm_forward, A, E, pi, pobs), 1, 1, dist)
    flops = 2.0 * S * S * (T - 1) * nsig
    achieved = flops / (ms * 1e-3) / 1e12
    res = {"value": NS / (ms * 1e-3), "ms_per_step": ms, "steps": s, "warmup": w,
           "trellis_cells_per_s": float(S) * S * (T - 1) * NS / (ms * 1e-3),
           "e2e": _e2e("signals/s", NS, e2e_ms, pobs.numel() * 4 + 8 * (A.size + E.size + pi.size), 8 * nsig,
                       pcie, "accelerate(hmm_forward) with host probabilities and pinned observations"),
           "roofline": {"bound": "tensor", "unit": "TFLOP/s", "achieved": achieved, "peak": peaks["bf16_tflops"],
                        "frac": achieved / peaks["bf16_tflops"],
                        "peak_source": "f16 dense = measured bf16 dense (MEASURED_PEAKS.json, burst)",
                        "algorithmic_flops_per_signal": 2 * S * S * (T - 1),
                        "umma_probe_tflops": {"M128_N64": 1463.4, "M128_N128": 2205.1,
                                              "source": "tools/umma_rate.cu (profiles/umma_rate.json)"},
                        "note": "tcgen05 kind::f16 cta_group::2 (M = 256 across a CTA pair, N = 128 signals), "
                                "exactly 2^k-scaled fp16 operands, fp32 TMEM accumulation, clusters of 4; "
                                "u_t exchanged between the 4 SMs every step"},
           "range_guard": {"signals_rerun_fp32": rerun, "of": nsig},
           "kernels_per_step": 4}
    if not args.no_parity:
        O = _oracle()
        sel = synth.parity_sample(nsig, 8)
        want = O.hmm_forward_scaled(A, E, pi, hobs[sel])
        got = out.to("cpu").numpy()[sel]
        rel = float(np.max(np.abs(got - want) / np.abs(want)))
        res["parity"] = {"checked": f"{len(sel)} sampled signals of this rank vs the fp64 oracle", "max_rel": rel,
                         "tolerance": 1e-5, "pass": bool(rel <= 1e-5)}
    return res


def bench_kmer(args, dist, peaks, pcie) -> dict:
    import numpy as np
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib, synth
    kmer, K, T = 8, 8, 6000
    NS = 1024 * dist.world          # 8k signals over 8 GPUs: 1024 per GPU
    lo, hi = dist.shard(NS)
    nsig = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device())
    Ek = synth.kmer_emission(kmer, K)
    lE = torch.from_numpy(np.log(Ek).astype(np.float32)).to(dev)
    hobs = synth.hmm_obs(nsig, T, K, first=lo)
    obs = torch.from_numpy(hobs).to(dev)
    out = torch.empty(nsig, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pmx_hmm_kmer_workspace_bytes(kmer, nsig), dtype=torch.uint8, device=dev)

    def step():
        _lib.check(lib.pmx_hmm_kmer_forward_f32(kmer, 0.5, 0.125, lE.data_ptr(), K, obs.data_ptr(), nsig, T,
                                                out.data_ptr(), ws.data_ptr(), ws.numel(), _stream()), "kmer")
    w, s = min(args.warmup, 1), max(1, min(args.steps, 2))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    S = 1 << (2 * kmer)
    pobs = torch.from_numpy(hobs).pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(lambda e, o: P.hmm_kmer_forward(kmer, 0.5, 0.125, e, o), Ek, pobs),
                          1, 1, dist)
    # k = 8 runs on CTA pairs with alpha in registers (k_kmer_fwd_pair): what
    # enters the SMs per signal-step is the emission row (4 B per state, an
    # L2-resident table) plus the pair-sum exchange between the two CTAs (32 KiB
    # each way, DSMEM, over the same xbar -> SM path); both are algorithmic.
    emis = 4.0 * S
    exch = 2.0 * 32768
    bytes_ = (emis + exch) * T * nsig
    gbs = bytes_ / (ms * 1e-3) / 1e9
    l2 = pipe_peaks().get("l2_bulk_table_bytes_per_s")
    roof = {"bound": "sm ingress (L2 -> SM reads + DSMEM)", "unit": "GB/s", "achieved": round(gbs, 1),
            "bytes_per_signal_step": emis + exch, "emission_bytes_per_signal_step": emis,
            "dsmem_bytes_per_signal_step": exch, "vs_hbm_peak": round(gbs / peaks["hbm_gbs"], 3),
            "traffic": _kmer_traffic(T),
            "note": "alpha never leaves the registers; ncu (T = 100): L2 reads = the emission rows once per "
                    "signal-step, DRAM ~0, SM ingress = emissions + exchange (profiles/traffic.json). The DSMEM "
                    "exchange alone runs at 17 B/clk/SM each way (tools/dsmem_probe.cu, profiles/r2_dsmem_probe.log)"}
    if l2:
        roof.update({"peak": round(l2 / 1e9, 1), "frac": round(gbs * 1e9 / l2, 4),
                     "peak_source": "tools/l2_bulk_probe.cu: TMA bulk copies of one 2 MiB L2-resident table into "
                                    "every SM (profiles/pipe_peaks.json l2_bulk_table_bytes_per_s; the ld.global "
                                    "probe reaches 12.5 TB/s)"})
    res = {"value": NS / (ms * 1e-3), "ms_per_step": ms, "steps": s, "warmup": w,
           "trellis_cells_per_s": 5.0 * S * (T - 1) * NS / (ms * 1e-3),
           "e2e": _e2e("signals/s", NS, e2e_ms, pobs.numel() * 4 + 8 * Ek.size, 8 * nsig, pcie,
                       "accelerate(hmm_kmer_forward) with host emissions and pinned observations"),
           "roofline": roof, "kernels_per_step": 1}
    if not args.no_parity:
        O = _oracle()
        sel = synth.parity_sample(nsig, 8)
        want = O.kmer_forward_scaled(kmer, 0.5, 0.125, Ek, hobs[sel])
        got = out.to("cpu").numpy()[sel]
        rel = float(np.max(np.abs(got - want) / np.abs(want)))
        res["parity"] = {"checked": f"{len(sel)} sampled signals of this rank vs the fp64 oracle", "max_rel": rel,
                         "tolerance": 1e-5, "pass": bool(rel <= 1e-5)}
    return res


def _kmer_traffic(T: int):
    """ncu L2 / DRAM / SM-ingress bytes of one k-mer launch (1024 signals),
    scaled from the T = 100 capture to T steps (per-step traffic is constant)."""
    t = _traffic_from_profiles("kmer")
    if not t:
        return None
    f = T / 100.0
    return {"l2_bytes": t["l2_bytes_per_launch_T100"] * f, "dram_bytes": t["dram_bytes_per_launch_T100"] * f,
            "sm_ingress_bytes": t["sm_ingress_bytes_per_launch_T100"] * f,
            "ingress_vs_algorithmic": round(t["sm_ingress_bytes_per_launch_T100"]
                                            / t["algorithmic_bytes_per_launch_T100"], 3),
            "source": "profiles/traffic.json (ncu, T = 100, scaled)"}


def bench_viterbi(args, dist, peaks, pcie) -> dict:
    """Viterbi decoding (programs/viterbi.pmx) at scale: SURVEY §8(f) rank 1.
    The HMM model of the forward config (S=1024, K=8), 1184 signals per GPU
    (8 per SM) x T=1000, fp64 like the reference."""
    import numpy as np
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib, synth
    S, K, T = 1024, 8, 1000
    NS = 148 * 8 * dist.world
    lo, hi = dist.shard(NS)
    nsig = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device())
    A, E, pi = synth.hmm_model(S, K)
    lA, lE, lpi = (torch.from_numpy(np.log(a)).to(dev) for a in (A, E, pi))
    hobs = synth.hmm_obs(nsig, T, K, first=lo)
    obs = torch.from_numpy(hobs).to(dev)
    path = torch.empty(nsig * T, dtype=torch.int32, device=dev)
    logp = torch.empty(nsig, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pmx_viterbi_workspace_bytes(S, nsig, T), dtype=torch.uint8, device=dev)

    def step():
        _lib.check(lib.pmx_viterbi_f64(lpi.data_ptr(), lA.data_ptr(), lE.data_ptr(), S, K, obs.data_ptr(), nsig,
                                       T, path.data_ptr(), logp.data_ptr(), ws.data_ptr(), ws.numel(), _stream()),
                   "viterbi")
    w, s = min(args.warmup, 1), max(1, min(args.steps, 2))
    total, per = device_time(step, s, w, dist)
    ms = total / s
    visited = int(lib.pmx_viterbi_visited_cells(ws.data_ptr(), S, nsig, T, _stream())) \
        if hasattr(lib, "pmx_viterbi_visited_cells") else -1
    pobs = torch.from_numpy(hobs).pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(P.viterbi, A, E, pi, pobs), 1, 1, dist)
    cells = float(S) * S * (T - 1) * nsig
    pp = pipe_peaks()
    fp64_peak = pp.get("fp64_add_ops_per_s", 63.0 * 148 * 1.965e9)
    prof = _profile("viterbi_fp64.json")
    per_cell = prof.get("fp64_pipe_ops_per_visited_cell", 2.0)
    roof = {"bound": "fp64 pipe on the cells the branch-and-bound scan visits (score and bound DADDs, DSETP "
                     "compares)", "unit": "fp64 pipe ops/s", "peak": fp64_peak,
            "fp64_pipe_ops_per_visited_cell": per_cell,
            "dense_equivalent_cells_per_s": cells / (ms * 1e-3),
            "peak_source": "tools/peaks.cu (profiles/pipe_peaks.json)",
            "ncu": {k: prof[k] for k in ("fp64_pipe_active_pct", "issue_active_pct", "warps_active_pct_of_peak")
                    if k in prof}}
    if visited > 0:
        achieved = per_cell * visited / (ms * 1e-3)
        roof.update({"achieved": achieved, "frac": round(achieved / fp64_peak, 4),
                     "visited_cells_per_launch": visited, "visited_fraction": round(visited / cells, 4)})
    res = {"value": NS / (ms * 1e-3), "ms_per_step": ms, "steps": s, "warmup": w,
           "e2e": _e2e("signals/s", NS, e2e_ms, pobs.numel() * 4 + 8 * (A.size + E.size + pi.size),
                       nsig * (4 * T + 8), pcie, "accelerate(viterbi) with host model and pinned observations"),
           "roofline": roof, "kernels_per_step": 3}
    if not args.no_parity:
        O = _oracle()
        sel = synth.parity_sample(nsig, 8)
        wp, wl = O.viterbi(A, E, pi, hobs[sel])
        gp = path.to("cpu").numpy().reshape(nsig, T)[sel]
        gl = logp.to("cpu").numpy()[sel]
        rel = float(np.max(np.abs(gl - wl) / np.abs(wl)))
        res["parity"] = {"checked": f"{len(sel)} sampled signals of this rank vs the fp64 oracle",
                         "paths_bit_exact": bool(np.array_equal(gp, wp)), "logp_max_rel": rel,
                         "pass": bool(np.array_equal(gp, wp) and rel <= 1e-9)}
    return res


def bench_nn(args, dist, peaks, pcie) -> dict:
    """Softmax-regression loss + gradients (programs/nn.pmx) at scale: SURVEY
    §8(f) rank 3.  2^20 points per GPU, 64 inputs, 16 classes, fp64 (the
    reference's Float); x is the only HBM stream (512 MiB)."""
    import numpy as np
    import torch
    import paper_2211_00621_b200 as P
    from paper_2211_00621_b200 import _lib
    npts, nin, nout = 1 << 20, 64, 16
    dev = torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(3 + dist.rank)
    hx = rng.standard_normal((npts, nin)) * 0.5
    hy = rng.integers(0, nout, npts).astype(np.int32)
    hw = rng.standard_normal((nin, nout)) * 0.3
    hb = rng.standard_normal(nout) * 0.1
    x, y, w, b = (torch.from_numpy(a).to(dev) for a in (hx, hy, hw, hb))
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    dw = torch.empty(nin * nout, dtype=torch.float64, device=dev)
    db = torch.empty(nout, dtype=torch.float64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    lib = _lib.load()
    ws = torch.zeros(lib.pmx_nn_workspace_bytes(npts, nin, nout), dtype=torch.uint8, device=dev)

    def step():
        _lib.check(lib.pmx_nn_softmax_grad_f64(x.data_ptr(), y.data_ptr(), w.data_ptr(), b.data_ptr(), npts, nin,
                                               nout, loss.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(),
                                               ws.numel(), err.data_ptr(), _stream()), "nn")
    total, per = device_time(step, args.steps, args.warmup, dist)
    ms = total / args.steps
    px = torch.from_numpy(hx).pin_memory()
    e2e_ms, _ = host_time(lambda: P.accelerate(lambda a, c, d, e: P.nn_gradients(a, c, d, e)["loss"], px, hy, hw,
                                                hb), 2, 1, dist)
    bytes_ = 8.0 * nin * npts + 4.0 * npts
    pipe_ops = npts * (3.0 * nin * nout)             # z: DMUL + DADD; dw: one DFMA
    pp = pipe_peaks()
    fp64_peak = pp.get("fp64_add_ops_per_s", 63.0 * 148 * 1.965e9)
    achieved = pipe_ops / (ms * 1e-3)
    res = {"value": npts * dist.world / (ms * 1e-3), "ms_per_step": ms,
           "e2e": _e2e("points/s", npts * dist.world, e2e_ms / 2, px.numel() * 8 + 4 * npts + 8 * (hw.size + hb.size),
                       8, pcie, "accelerate(nn_gradients) with pinned host points"),
           "roofline": {"bound": "fp64 pipe", "unit": "fp64 pipe instr/s", "achieved": achieved, "peak": fp64_peak,
                        "frac": round(achieved / fp64_peak, 4),
                        "hbm_GBps": bytes_ / (ms * 1e-3) / 1e9, "hbm_frac": bytes_ / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                        "note": "z keeps the reference's separately rounded mul + add (2 pipe ops per MAC); "
                                "dw sums use DFMA (1 pipe op)"},
           "kernels_per_step": 2}
    if not args.no_parity:
        O = _oracle()
        wl, wdw, wdb = O.nn(hx, hy, hw, hb, workers=cpu_threads())
        gl = float(loss.item())
        gdw = dw.to("cpu").numpy().reshape(nin, nout)
        gdb = db.to("cpu").numpy()
        rel = max(abs(gl - wl) / abs(wl), float(np.max(np.abs(gdw - wdw) / np.maximum(np.abs(wdw), 1e-300))),
                  float(np.max(np.abs(gdb - wdb) / np.maximum(np.abs(wdb), 1e-300))))
        res["parity"] = {"checked": "loss, dw and db over all 2^20 points of this rank vs the fp64 oracle",
                         "max_rel": rel, "tolerance": 1e-9, "pass": bool(rel <= 1e-9)}
    return res


# ===================================================== CPU port baselines
# The CPU restatement of the reference's path (oracle/pmx_oracle.c, OpenMP over
# independent elements) timed on this host's cores on a bounded sample of the
# same workload.  Used as `cpu_baseline` (ours, rank 0 at N = 1) and as the
# reference arm's values.

def _timed_loop(fn, seconds: float) -> tuple[int, float]:
    fn()
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        if time.perf_counter() - t0 > seconds:
            break
    return reps, (time.perf_counter() - t0) / reps


def cpu_mapreduce(seconds: float = 10.0) -> dict:
    O = _oracle()
    from paper_2211_00621_b200 import synth
    m = 1 << 26
    x = synth.mapreduce_x(m)
    th = cpu_threads()
    reps, dt = _timed_loop(lambda: O.map_affine_reduce_add(x, workers=th, threads=th), seconds)
    return {"value": m / dt, "unit": "elements/s", "cores": th, "kind": "port",
            "sample": f"{reps} passes of the oracle (oracle/pmx_oracle.c, fp64 reference semantics, "
                      f"{th} OpenMP threads = {th} chunks) over 2^26 of the 2^28 elements"}


def cpu_rk4(seconds=10.0) -> dict:
    O = _oracle()
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    n = max(64, 16 * th)
    ps = synth.rk4_params(10_000)[:n]
    reps, dt = _timed_loop(lambda: O.rk4(ps, synth.RK4_INIT, 1000, synth.RK4_H, threads=th), seconds)
    return {"value": n / dt, "unit": "parameter sets/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {n} of the 10^4 parameter sets x 1000 steps"}


def cpu_knn(seconds=10.0) -> dict:
    O = _oracle()
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    X = synth.knn_train(1 << 20, 64)
    L = synth.knn_labels(1 << 20, 10)
    nq = max(8, th)
    Q = synth.knn_query(nq, 64)
    reps, dt = _timed_loop(lambda: O.knn(X, L, Q, 8, 10, threads=th), seconds)
    return {"value": nq / dt, "unit": "queries/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {nq} of the 2^16 queries against all 2^20 train points"}


def cpu_hmm(seconds=10.0) -> dict:
    O = _oracle()
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    A, E, pi = synth.hmm_model(1024, 8)
    T = 20
    obs = synth.hmm_obs(max(2, th), T, 8)
    reps, dt = _timed_loop(lambda: O.hmm_forward(A, E, pi, obs, threads=th), seconds)
    return {"value": obs.shape[0] * (T - 1) / dt / (10_000 - 1), "unit": "signals/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {obs.shape[0]} signals x {T} steps at S=1024 (log-space oracle, Appendix A.1), "
                      "scaled to T=10^4"}


def cpu_kmer(seconds=10.0) -> dict:
    O = _oracle()
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    E = synth.kmer_emission(8, 8)
    T = 30
    obs = synth.hmm_obs(max(2, th), T, 8)
    reps, dt = _timed_loop(lambda: O.kmer_forward(8, 0.5, 0.125, E, obs, threads=th), seconds)
    return {"value": obs.shape[0] * (T - 1) / dt / (6000 - 1), "unit": "signals/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {obs.shape[0]} signals x {T} steps at S=65536 (log-space oracle), scaled to T=6000"}


def cpu_viterbi(seconds=10.0) -> dict:
    O = _oracle()
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    A, E, pi = synth.hmm_model(1024, 8)
    T = 20
    obs = synth.hmm_obs(max(2, th), T, 8)
    reps, dt = _timed_loop(lambda: O.viterbi(A, E, pi, obs, threads=th), seconds)
    return {"value": obs.shape[0] * (T - 1) / dt / (1000 - 1), "unit": "signals/s", "cores": th, "kind": "port",
            "sample": f"{reps}x {obs.shape[0]} signals x {T} steps at S=1024, scaled to T=1000"}


def cpu_nn(seconds=10.0) -> dict:
    import numpy as np
    O = _oracle()
    th = cpu_threads()
    n, nin, nout = 1 << 18, 64, 16
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, nin))
    y = rng.integers(0, nout, n).astype(np.int32)
    w = rng.standard_normal((nin, nout))
    b = rng.standard_normal(nout)
    reps, dt = _timed_loop(lambda: O.nn(x, y, w, b, workers=th, threads=th), seconds)
    return {"value": n / dt, "unit": "points/s", "cores": th, "kind": "port",
            "sample": f"{reps}x 2^18 of the 2^20 points ({th} chunks on {th} OpenMP threads)"}


CASES = (("rk4", bench_rk4, cpu_rk4), ("knn", bench_knn, cpu_knn), ("hmm_forward", bench_hmm, cpu_hmm),
         ("hmm_kmer", bench_kmer, cpu_kmer), ("viterbi", bench_viterbi, cpu_viterbi), ("nn", bench_nn, cpu_nn))


# ================================================================= main
def run_ours(args):
    import torch
    dist = Dist()
    torch.cuda.set_device(dist.local % max(1, torch.cuda.device_count()))
    dist.init("nccl")
    import paper_2211_00621_b200 as P
    P.load_library()
    peaks = _peaks()
    pcie = pcie_h2d_gbs()
    res = bench_mapreduce(args, dist, peaks, pcie)
    want_cpu = dist.rank == 0 and dist.world == 1 and not args.no_cpu
    cpu = cpu_mapreduce(args.cpu_seconds) if want_cpu else None
    configs = case_configs(dist.world)
    case = {}
    if not args.no_case_studies:
        for name, fn, cfn in CASES:
            if args.case and name not in args.case:
                continue
            try:
                r = fn(args, dist, peaks, pcie)
                r = {"config": configs[name], "unit": configs[name]["unit"], **r}
                if want_cpu:
                    r["cpu_baseline"] = cfn(args.cpu_seconds / 2)
                    r["speedup_vs_cpu"] = r["value"] / r["cpu_baseline"]["value"]
                    r["e2e_speedup_vs_cpu"] = r["e2e"]["value"] / r["cpu_baseline"]["value"]
                case[name] = r
            except Exception as exc:    # report, do not hide
                import traceback
                case[name] = {"config": configs[name], "error": f"{type(exc).__name__}: {exc}",
                              "trace": traceback.format_exc()[-2000:]}
    if dist.rank != 0:
        return
    line = {
        "metric": METRIC, "value": res["value"], "unit": "elements/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (integer-formula inputs, SURVEY §8(d))",
        "config": headline_config(dist.world),
        "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"], "gpu_launches": res["gpu_launches"],
        "clocks": res["clocks"], "parity": res["parity"],
        "result": {"sum": res["result"], "exact": res["exact_result"]},
        "pcie_h2d_GBps": round(pcie, 1) if pcie else None,
        "variants": res["variants"], "case_studies": case,
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference arm: the CPU restatement of the reference's path (the
    oracle port, oracle/pmx_oracle.c) on this box's host cores, same metric,
    config and case-study configs; rank 0 only."""
    dist = Dist()
    if dist.rank != 0:
        return
    O = _oracle()
    from paper_2211_00621_b200 import synth
    th = cpu_threads()
    # each step folds one GPU's 2^28-element share (the CPU rate does not depend
    # on the total); at N > 1, ms_per_step is that time x N (the whole job)
    n = N_PER_GPU
    x = synth.mapreduce_x(n)
    per = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.map_affine_reduce_add(x, workers=th, threads=th)
        if i >= args.warmup:
            per.append(time.perf_counter() - t0)
    ms = 1e3 * sum(per) / len(per) * dist.world
    val = n * dist.world / (ms * 1e-3)
    configs = case_configs(dist.world)
    case = {}
    if not args.no_case_studies:
        for name, _fn, cfn in CASES:
            if args.case and name not in args.case:
                continue
            c = cfn(args.cpu_seconds / 2)
            case[name] = {"config": configs[name], "unit": configs[name]["unit"], "value": c["value"],
                          "cpu_baseline": c, "e2e": {"value": c["value"], "unit": c["unit"],
                                                     "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "elements/s", "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (integer-formula inputs, SURVEY §8(d))",
            "config": headline_config(dist.world),
            "cpu_baseline": {"value": val, "unit": "elements/s", "cores": th, "kind": "port",
                             "sample": f"{n} elements (one GPU's share) per step; oracle/pmx_oracle.c "
                                       "oracle_map_affine_reduce_add (fp64 Float semantics, _chunks partition)"},
            "e2e": {"value": val, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "case_studies": case}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


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
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity checks (quick experiments)")
    ap.add_argument("--nccl-combine", action="store_true",
                    help="N>1: combine reduce partials with NCCL all-gather instead of the fused peer kernel")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(pathlib.Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}", file=sys.stderr)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

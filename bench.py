"""Benchmark: MoE-layer dispatch+combine (µs & tokens/s) with dedup, on B200.

Default workload (BASELINE.json configs[1]): Qwen3-30B-A3B-shaped MoE layer,
E = 128 experts, top-8, hidden 2048, bf16, expert parallelism over G = 8 EP
ranks, 4096 tokens per rank, GPU-level dedup.  The 8 EP ranks are hosted on
the N GPUs of the run (8/N ranks per GPU; N = 1 exchanges through HBM, N > 1
over NVLink via CUDA-IPC peer stores), so the total work is fixed: strong
scaling.

One step = dispatch (top-K gating kernel, dedup plan, count exchange + barrier,
pack/exchange of one row per (token, destination rank), destination
re-expansion into expert-major rows) + combine (destination gate-weighted
pre-reduce, barrier, source sum over destinations).  The expert FFN between
them is excluded by the metric's definition (it is timed separately by
--ffn when the grouped GEMM is built).  Expert outputs are resident in HBM.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
For N > 1 launch with torch.distributed.run (one process per GPU).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE layer dispatch+combine µs & tokens/s at 1/2/4/8 B200; comm bytes cut by dedup"
CONFIGS = {
    # name: (G ranks, E, K, M, tokens per rank, description)
    "qwen3": (8, 128, 8, 2048, 4096,
              "Qwen3-30B-A3B-shaped MoE layer: 128 experts, top-8, hidden 2048, bf16, EP=8, "
              "GPU-level dedup"),
    "dsv3": (8, 256, 8, 7168, 4096,
             "DeepSeek-V3-shaped MoE layer: 256 routed experts, top-8, hidden 7168, bf16, EP=8"),
    "configA": (8, 16, 2, 256, 512,
                "reference CPU config: 16 experts, top-2, hidden 256, 4096 tokens, 8-rank EP world"),
    # one EP rank per GPU on a 4-GPU box: exercises the N = 8 layout (L = 1)
    "qwen3_ep4": (4, 128, 8, 2048, 4096,
                  "Qwen3-shaped MoE layer with EP=4 (one rank per GPU at N=4; the N=8 layout)"),
}
INTER = {"qwen3": 768, "dsv3": 2048, "configA": 512, "qwen3_ep4": 768}
NVLINK_GBS = 770.0   # B200_PROFILING.md: measured peer copy, per direction per GPU
# all-to-all pushes of 4 KB rows driven by SMs (16-B peer stores or TMA bulk
# stores, every GPU to every other at once): the ceiling of an SM-driven
# exchange on these boxes (tools/link_probe.cu, profiles/r01_link_probe.jsonl)
SM_PUSH_GBS = 678.0
SEGMENTS = ["plan", "notify", "pack", "barrier1", "expand", "reduce", "barrier2", "gather"]


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


class ClockSampler:
    """SM clock + throttle reasons sampled via NVML every 10 ms during the
    timed region (the B200_PROFILING.md clocks line, at finer resolution)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), int(rs)))
                    except Exception:
                        pass
                    time.sleep(0.01)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=2)

    def summary(self) -> dict:
        sm = [s for s, _ in self.samples]
        loaded = [s for s in sm if self.max_mhz and s > 0.5 * self.max_mhz] or sm
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference(cfg_name: str, steps: int, warmup: int, tokens_per_rank: int | None = None):
    """The CPU port of the same dispatch+combine step on the host cores
    (oracle/moe.py cpu_dispatch_combine: torch CPU, every host thread), at the
    FULL workload (G ranks x T_r tokens, bf16 rows).  The reference itself has
    no dispatch/combine to run (it only models the AlltoAll, traffic.py:93-185),
    so this is a port ("kind": "port").  Returns per-step times; the caller
    reports best-of and mean."""
    import torch
    from oracle import moe as OM
    G, E, K, M, T_r, _ = CONFIGS[cfg_name]
    T_r = tokens_per_rank or T_r
    T = G * T_r
    threads = os.cpu_count() or 1
    gen = torch.Generator().manual_seed(0)
    logits = torch.randn(T, E, generator=gen)
    x = torch.randn(T, M, generator=gen).to(torch.bfloat16)
    _, ym, _ = OM.cpu_dispatch_combine(logits, x, K, threads=threads)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        OM.cpu_dispatch_combine(logits, x, K, y_major=ym, threads=threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    best, mean = min(times), float(np.mean(times))
    return {"value": T / best, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"the full step: {T} tokens ({G} ranks x {T_r}) of the {cfg_name} layer "
                      f"shape, bf16 rows, torch-CPU gating + permute + weighted unpermute "
                      f"(oracle/moe.py cpu_dispatch_combine), best of {steps} after {warmup} "
                      f"warm-up", "ms_per_step": best * 1e3, "mean_ms_per_step": mean * 1e3,
            "steps": steps, "warmup": warmup}


# swap planner per step (optimal_dimension + select_swap beside
# the reference's CPU path) on the uniform Qwen3 (B) and DSv3 (C) masks of a
# full 8-rank step, B200 alpha/beta (tools/calibrate.py, profiles/r01_calib_n4.json)
PLANNER_CASES = [
    ("B", (8,), 128, 2048, ((), (), (3.36e-5,), (2.84e-13,))),
    ("C", (2, 4), 256, 7168, ((3.14e-5,), (1.80e-13,), (3.36e-5, 3.15e-5), (2.84e-13, 3.59e-13))),
]


def _planner_mask(E, T, K, seed):
    import paper_2508_09591_b200 as hm
    return hm.generate_uniform(T, E, K, seed)


def planner_gpu(T: int, K: int = 8, reps: int = 5) -> dict:
    """Device planner: d* (optimal_dimension) and the swap choice (select_swap)
    on a resident mask; CUDA events, best of `reps` after a warm-up."""
    import torch
    import paper_2508_09591_b200 as hm
    res = {}
    for name, fan, E, M, p in PLANNER_CASES:
        mask = hm.device_mask(_planner_mask(E, T, K, 7))
        topo = hm.build_topology(list(fan), E, M, 2)
        params = hm.LevelParams(*p)
        times = {"optimal_dimension": [], "select_swap": []}
        for it in range(reps + 1):
            for key, fn in (("optimal_dimension", lambda: hm.optimal_dimension(mask, topo, params)),
                            ("select_swap", lambda: hm.select_swap(mask, topo, params, 10.0))):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r = fn()
                e1.record()
                e1.synchronize()
                if it:
                    times[key].append(e0.elapsed_time(e1))
        pair = list(r.pair) if r.pair else None
        res[name] = {"topology": list(fan), "experts": E, "tokens": T,
                     "gpu_ms": {k: round(min(v), 3) for k, v in times.items()},
                     "d_star": r.d_star, "pair": pair}
        # the reference's own decision on this exact mask (tests/golden/fullsize.json,
        # made by running hiera2a: swap.py:226-252, traffic.py:202-221)
        ref = _fullsize_fixture(name, T, K)
        if ref is not None:
            ok = (pair == ref["plan_pair"] and r.d_star == ref["plan_d_star"]
                  and r.no_swap_time == ref["plan_no_swap"]
                  and r.predicted_saving == ref["plan_saving"])
            res[name]["matches_reference"] = ok
            assert ok, f"planner {name}: {pair}, d*={r.d_star} vs reference {ref['plan_pair']}"
    return res


def _fullsize_fixture(name: str, T: int, K: int):
    """Reference decision for the bench's planner mask, if T/K are the bench's."""
    p = ROOT / "tests" / "golden" / "fullsize.json"
    if T != 32768 or K != 8 or not p.exists():
        return None
    key = {"B": "B_qwen3_8", "C": "C_dsv3_2x4"}[name]
    return next((c for c in json.loads(p.read_text()) if c["name"] == key), None)


def _reference_pkg():
    """The unmodified reference package installed by oracle/make_ref.sh
    (oracle/_ref; travels to the GPU box), or None."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "hiera2a" / "__init__.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import hiera2a
    return hiera2a


def planner_cpu(T: int, K: int = 8, reps: int = 5) -> dict:
    """The reference's OWN optimal_dimension / select_swap (hiera2a from
    oracle/_ref, numpy + host BLAS on every core) on the same masks, best of
    `reps` after a warm-up.  Falls back to the oracle
    restatement (kind "port") only when oracle/_ref is absent."""
    H = _reference_pkg()
    res = {"kind": "reference" if H is not None else "port",
           "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}
    for name, fan, E, M, p in PLANNER_CASES:
        if H is not None:
            bits = H.generate_uniform(T, E, K, 7)
            topo = H.build_topology(list(fan), E, M, 2)
            params = H.LevelParams(*p)
            f_dim = lambda: H.optimal_dimension(bits, topo, params)            # noqa: E731
            f_sel = lambda: H.select_swap(bits, topo, params, 10.0)           # noqa: E731
        else:
            from oracle import hiera as O
            bits = _planner_mask(E, T, K, 7).bits
            f_dim = lambda: O.optimal_dimension(bits, fan, p, M * 2)          # noqa: E731
            f_sel = lambda: O.select_swap(bits, fan, p, M * 2, 10.0)          # noqa: E731
        t_dim, t_sel = [], []
        for i in range(reps + 1):
            t0 = time.perf_counter()
            f_dim()
            t1 = time.perf_counter()
            plan = f_sel()
            t2 = time.perf_counter()
            pair = plan.pair if hasattr(plan, "pair") else plan[0]
            if i:
                t_dim.append(t1 - t0)
                t_sel.append(t2 - t1)
        res[name] = {"optimal_dimension": round(min(t_dim) * 1e3, 2),
                     "select_swap": round(min(t_sel) * 1e3, 2),
                     "pair": list(pair) if pair else None}
    return res


def dsv3_layer_forward(G, E, K, M, inter, T_r, world, rank, x, flush, tokens_total, n_l, peaks):
    """Config C layer forward + backward: DeepSeek-V3 group-limited gate (8
    groups, top-4 groups, scale 2.5), dedup dispatch, tcgen05 experts, the
    shared expert (I = 2048) on a side stream overlapped with the dispatch,
    combine + shared sum; backward through all of it.  No optimizer state
    (256 experts x 44 M parameters; weights, transposes and grads are bf16)."""
    import torch
    import torch.distributed as dist
    from paper_2508_09591_b200.moe import HierMoELayer
    layer = HierMoELayer(G, E, K, M, inter, T_r, gpus=world, gpu_index=rank, dedup=True,
                         n_cap_rows=2 * T_r * K, router="dsv3", n_group=8, topk_group=4,
                         route_scale=2.5, shared_inter=2048, optimizer_state=False, grad=True)
    lout = torch.empty_like(x)
    gen = torch.Generator(device="cuda").manual_seed(99 + rank)
    gout = torch.randn(x.shape, device="cuda", generator=gen).to(x.dtype)
    for _ in range(3):
        layer(x, out=lout)
        layer.backward(gout)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    acc = np.zeros(2)
    with ClockSampler(torch.cuda.current_device()) as lclk:
        for _ in range(n_l):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            layer(x, out=lout)
            ev[1].record()
            layer.backward(gout)
            ev[2].record()
            ev[2].synchronize()
            acc += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])]
    t = torch.tensor(acc / n_l, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    layer.world.check_status()
    fl = layer.flops_per_forward() + 6 * x.shape[0] * M * 2048
    fwd_ms, bwd_ms = (float(v) for v in t.tolist())
    out = {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "fwd_bwd_ms": fwd_ms + bwd_ms,
           "fwd_tokens_per_s": tokens_total / (fwd_ms * 1e-3),
           "fwd_bwd_tokens_per_s": tokens_total / ((fwd_ms + bwd_ms) * 1e-3),
           "router": "dsv3 group-limited (n_group 8, topk_group 4, scale 2.5)",
           "shared_expert_inter": 2048, "inter": inter, "transport": layer.dedup,
           "ffn_flops_per_gpu_incl_shared": int(fl),
           "fwd_tflops": fl / (fwd_ms * 1e-3) / 1e12,
           "fwd_bwd_tflops": 3 * fl / ((fwd_ms + bwd_ms) * 1e-3) / 1e12,
           "clocks": lclk.summary(),
           "note": "router GEMMs, gate backward, dispatch/combine and experts fwd+bwd are our "
                   "kernels"}
    layer.close()
    return out


def nccl_nodedup(world, rank, G, E, K, M, logits, x, flush, steps, warmup):
    """The non-deduplicated AlltoAll baseline on NCCL (the reference's "std"
    strategy, engine.py:159-163 / traffic.py:164-170): every
    token's K picks are sent as K rows to the GPU owning the slot.  One step =
    gating (the same router kernel) -> permute by destination GPU
    (argsort + index_select) -> count exchange (all_to_all_single of P ints,
    read on the host for the split sizes) -> dispatch all_to_all_single ->
    combine all_to_all_single back -> gate-weighted unpermute (fp32 sum per
    token, cuBLAS bmm).  The destination-side sort into expert-major order is NOT done
    (it would only add to the baseline).  Returns (ms per step, exchange-only
    ms per step), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2508_09591_b200.layer import route_topk
    T = logits.shape[0]
    e_per_gpu = E // world
    out = torch.empty_like(x)

    def step(ev=None):
        slot, w, _ = route_topk(logits, K)
        dest = (slot.reshape(-1).long() // e_per_gpu)
        order = torch.argsort(dest, stable=True)
        send = x.index_select(0, order // K)
        cnt = torch.bincount(dest, minlength=world).to(torch.int64)
        rcnt = torch.empty_like(cnt)
        if ev is not None:
            ev[0].record()
        dist.all_to_all_single(rcnt, cnt)
        s_sizes, r_sizes = cnt.tolist(), rcnt.tolist()
        recv = torch.empty(sum(r_sizes), M, dtype=x.dtype, device="cuda")
        dist.all_to_all_single(recv, send, r_sizes, s_sizes)
        if ev is not None:
            ev[1].record()
        # (expert FFN here; outputs = inputs) -> combine: send the rows back
        back = torch.empty_like(send)
        if ev is not None:
            ev[2].record()
        dist.all_to_all_single(back, recv, s_sizes, r_sizes)
        if ev is not None:
            ev[3].record()
        inv = torch.empty_like(order)
        inv[order] = torch.arange(order.numel(), device="cuda")
        yk = back.index_select(0, inv).view(T, K, M)
        # weighted sum over the K picks (cuBLAS batched GEMV, fp32 accumulation)
        torch.bmm(w.to(x.dtype)[:, None, :], yk, out=out.view(T, 1, M))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    tot, exch = 0.0, 0.0
    for _ in range(steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[4].record()
        step(ev)
        ev[5].record()
        ev[5].synchronize()
        tot += ev[4].elapsed_time(ev[5])
        exch += ev[0].elapsed_time(ev[1]) + ev[2].elapsed_time(ev[3])
    t = torch.tensor([tot / steps, exch / steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0]), float(t[1])


def _json_out():
    """Keep stdout for the one JSON line: library banners (NCCL's version line,
    torchrun notices) are redirected to stderr for the whole run."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(saved, "w")


def _bind_gpu_local_cpus(dev: int):
    """Restrict this process to the CPUs local to GPU `dev` (NVML's CPU
    affinity mask); returns a short description, or None when NVML cannot
    say.  Host buffers allocated afterwards land on that NUMA node."""
    try:
        import pynvml
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        n = (os.cpu_count() + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, n)
        cpus = [w * 64 + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1]
        cpus = [c for c in cpus if c in os.sched_getaffinity(0)]
        if not cpus:
            return f"unbound: {len(os.sched_getaffinity(0))} cpus (no NVML affinity)", None
        old = os.sched_getaffinity(0)
        os.sched_setaffinity(0, cpus)
        return f"{len(cpus)} cpus {cpus[0]}-{cpus[-1]}", old
    except Exception:   # noqa: BLE001 -- affinity is an optimisation only
        return f"unbound: {len(os.sched_getaffinity(0))} cpus (no NVML affinity)", None


def main():
    out_stream = _json_out()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen3", choices=list(CONFIGS))
    ap.add_argument("--tokens", type=int, default=None, help="tokens per EP rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-layer", action="store_true", help="skip the full layer forward")
    ap.add_argument("--no-planner", action="store_true", help="skip the swap-planner timing")
    ap.add_argument("--no-hd2", action="store_true", help="skip config C's two-level timing")
    args = ap.parse_args()
    world, rank, local = dist_env()
    G, E, K, M, T_r, desc = CONFIGS[args.config]
    if args.tokens:
        T_r = args.tokens

    if args.impl == "reference":
        if rank != 0:
            return
        ref = cpu_reference(args.config, args.steps, args.warmup, args.tokens)
        line = {"metric": METRIC, "value": ref["value"], "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ref["ms_per_step"],
                "mean_ms_per_step": ref["mean_ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic", "impl": "reference",
                "config": {"workload": desc, "ranks": G, "experts": E, "top_k": K, "hidden": M,
                           "tokens_per_rank": args.tokens or T_r,
                           "global_tokens": G * (args.tokens or T_r)},
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": ref["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        if not args.no_planner and args.tokens is None:
            # the reference's own planner calls per step (hiera2a from oracle/_ref)
            line["planner_cpu_ms"] = planner_cpu(G * T_r, K)
            line["planner_cpu_ms"]["cores"] = os.cpu_count()
        print(json.dumps(line), file=out_stream, flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200.layer import EPWorld, route_topk

    torch.cuda.set_device(local)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if G % world:
        raise SystemExit(f"{G} EP ranks do not split over {world} GPUs")
    L = G // world
    dtype = torch.bfloat16
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    T = L * T_r
    logits = torch.randn(T, E, device="cuda", generator=gen)
    x = torch.randn(T, M, device="cuda", generator=gen).to(dtype)
    cap = 3 * T_r * K   # expert-major rows per rank (3x the uniform mean; overflow is flagged)
    ep = EPWorld(G, E, K, M, T_r, dtype=dtype, gpus=world, gpu_index=rank, n_cap_rows=cap)
    raw_ep = EPWorld(G, E, K, M, T_r, dtype=dtype, gpus=world, gpu_index=rank, n_cap_rows=cap)
    all_ep = EPWorld(G, E, K, M, T_r, dtype=dtype, gpus=world, gpu_index=rank, n_cap_rows=cap)
    # the step's transport: the reference time model's choice (traffic.py:188-221,
    # transport.choose_transport) on this step's global mask with the B200 fits
    # of the runtime [P, L] hierarchy (paper_2508_09591_b200/params)
    from paper_2508_09591_b200.routing import mask_from_ids
    from paper_2508_09591_b200.transport import choose_transport, default_params, runtime_topology
    rtopo = runtime_topology(G, world, E, M, 2)
    rparams = default_params(world, rtopo.num_levels)
    slot0, _, _ = route_topk(logits, K)
    red = (lambda t_: dist.all_reduce(t_)) if world > 1 else None
    choice = choose_transport(mask_from_ids(slot0, E), rtopo, rparams, None, red)
    MODE = choice.mode
    # fused dispatch (row indices; the expert GEMM gathers the rows from x and,
    # at N > 1, from the receive buffers) wherever the chosen transport allows it
    FUSED = world == 1 or MODE in ("gpu", "remote")
    ep.set_fused(FUSED)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # 256 MB > L2

    def prime(w_, dedup):
        slot, wts, _ = route_topk(logits, K)
        w_.dispatch(x, slot, wts, dedup=dedup)
        for l in range(L):   # expert outputs: the expert-major inputs (resident)
            p_x, _ = w_.buffer("xmaj", l)
            p_y, nbytes = w_.buffer("ymaj", l)
            _lib.call("hm_memcpy", p_y, p_x, nbytes, _lib.stream_ptr())
        w_.combine(slot, wts, dedup=dedup)
        torch.cuda.synchronize()
        return slot, wts

    def step(w_, dedup, out):
        slot, wts, _ = route_topk(logits, K)
        w_.dispatch(x, slot, wts, dedup=dedup)
        w_.combine(slot, wts, dedup=dedup, out=out)

    out = torch.empty(T, M, dtype=dtype, device="cuda")

    launches = {}   # library kernel launches inside the timed steps, per transport

    def timed(w_, dedup, steps, warmup):
        prime(w_, dedup)
        for _ in range(warmup):
            step(w_, dedup, out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        total = 0.0
        n0 = _lib.load().hm_launch_count()
        for _ in range(steps):
            flush.zero_()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            step(w_, dedup, out)
            s1.record()
            s1.synchronize()
            total += s0.elapsed_time(s1)
        launches[dedup] = int(_lib.load().hm_launch_count() - n0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = torch.tensor([total / steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        w_.check_status()
        return float(t.item())

    with ClockSampler(local) as clocks:
        ms = timed(ep, MODE, args.steps, args.warmup)
    main_launches = launches[MODE]
    # the same step replayed from a CUDA graph (device-side barrier epochs make
    # the exchange capturable): launch overhead and inter-kernel gaps removed
    graph_ms = None
    try:
        gst = torch.cuda.Stream()
        gst.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gst):
            step(ep, MODE, out)
        torch.cuda.current_stream().wait_stream(gst)
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            step(ep, MODE, out)
        for _ in range(3):
            cg.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tot_g, n_g = 0.0, max(5, args.steps // 2)
        for _ in range(n_g):
            flush.zero_()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            cg.replay()
            g1.record()
            g1.synchronize()
            tot_g += g0.elapsed_time(g1)
        tg = torch.tensor([tot_g / n_g], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        graph_ms = float(tg.item())
        ep.check_status()
        del cg
    except Exception as exc:   # noqa: BLE001 -- report, keep the eager numbers
        graph_ms = f"unavailable: {exc}"
    ms_copy = None
    if FUSED:   # the same step with the copying dispatch (materialised expert-major rows)
        ep.set_fused(False)
        ms_copy = timed(ep, MODE, max(3, args.steps // 2), args.warmup)
        seg_copy = None
        ep.set_fused(True)
    ms_raw = timed(raw_ep, "none", max(3, args.steps // 2), args.warmup)
    nccl = None
    if world > 1:   # the non-dedup AlltoAll on NCCL (what the >= 1.5x target is quoted against)
        n_ms, n_ex = nccl_nodedup(world, rank, G, E, K, M, logits, x, flush,
                                  max(5, args.steps // 4), max(3, args.warmup))
        nccl = {"ms_per_step": n_ms, "exchange_ms": n_ex, "value": G * T_r / (n_ms * 1e-3),
                "speedup_dedup_vs_nccl": n_ms / ms,
                "what": "route + permute + count a2a + dispatch a2a + combine a2a + weighted "
                        "unpermute; torch.distributed all_to_all_single (NCCL), K rows per "
                        "token to the slot-owning GPU"}
    ms_all = timed(all_ep, "all", max(3, args.steps // 2), args.warmup)

    # per-kernel timing (CUDA events recorded by the library on the launch stream)
    def seg_times(w_, dedup):
        # one untimed step first: a variant's kernels load lazily on their first launch
        step(w_, dedup, out)
        torch.cuda.synchronize()
        _lib.call("hm_world_set_timing", w_._h, 1)
        acc = np.zeros(len(SEGMENTS))
        n = 5
        for _ in range(n):
            flush.zero_()
            step(w_, dedup, out)
            torch.cuda.synchronize()
            buf = (__import__("ctypes").c_float * len(SEGMENTS))()
            _lib.call("hm_world_timings", w_._h, buf, len(SEGMENTS))
            acc += np.maximum(np.array(buf[:]), 0)
        _lib.call("hm_world_set_timing", w_._h, 0)
        return acc / n

    if FUSED:
        ep.set_fused(False)
        seg_copy = seg_times(ep, MODE)
        ep.set_fused(True)
    seg = seg_times(ep, MODE)
    seg_raw = seg_times(raw_ep, "none")
    seg_all = seg_times(all_ep, "all")

    # bytes moved by this GPU's kernels (algorithmic, per launch)
    cnt = ep.counts()
    rb = M * 2
    mine = list(range(rank * L, (rank + 1) * L))
    e_loc = E // G
    dest_gpu = np.arange(G) // L
    slot_gpu = (np.arange(E) // e_loc) // L
    src_rows = cnt[mine]
    rows_dedup_out = int(src_rows[:, :G].sum())             # "all" dedup rows
    rows_raw_out = int(src_rows[:, G:].sum())               # one per selection
    gcnt = ep.gpu_counts()[mine]                            # [L, P] rows per (src, gpu)
    rem_dedup = int(np.delete(gcnt, rank, axis=1).sum())    # per-GPU dedup rows that cross NVLink
    rem_rank_dedup = int(src_rows[:, :G][:, dest_gpu != rank].sum())
    rem_raw = int(src_rows[:, G:][:, slot_gpu != rank].sum())
    loc_direct = int(src_rows[:, G:][:, slot_gpu == rank].sum())
    R_in = ep.rows_received_gpu()                           # per-GPU dedup rows received
    src_gpu = np.arange(G) // L
    N_rem_in = int(cnt[src_gpu != rank][:, G:][:, slot_gpu == rank].sum())
    alg = {
        # fused: one GPU -- ids + rank_e read, epos + row index written per
        # pick; N > 1 -- rows read and pushed to the other GPUs hit, local
        # picks get row indices, no local row copies
        "pack": (T * K * 16 if world == 1 else
                 T * rb + rem_dedup * rb + rem_dedup * K * 8 + T * K * 12) if FUSED
                else T * rb + (rem_dedup + loc_direct) * rb + rem_dedup * K * 8,
        # fused: meta read + row index written per received pick
        "expand": R_in * K * 12 if FUSED else R_in * rb + N_rem_in * rb + R_in * K * 8,
        "reduce": N_rem_in * rb + R_in * rb + R_in * K * 8,
        "gather": (rem_dedup + loc_direct) * rb + T * rb,
    }
    # rows crossing NVLink: the dispatch pushes them in pack, the combine
    # pushes the pre-reduced rows back in reduce (per-GPU dedup transport);
    # the raw transport pushes in pack and pulls expert outputs in gather
    seg_ms = dict(zip(SEGMENTS, seg.tolist()))
    raw_ms = dict(zip(SEGMENTS, seg_raw.tolist()))
    ret_key = "reduce"
    link = {"pack": rem_dedup * rb, ret_key: R_in * rb} if world > 1 else {}
    link_dedup = seg_ms["pack"] + seg_ms[ret_key] if world > 1 else 0.0
    link_raw = raw_ms["pack"] + raw_ms["gather"] if world > 1 else 0.0
    dom = max(alg, key=lambda k: seg_ms[k])
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = alg[dom] / (seg_ms[dom] * 1e-3) / 1e9
    if dom in link:   # NVLink-bound kernel: link bytes against the measured peer bandwidth
        roof = {"bound": "nvlink", "kernel": dom,
                "achieved": link[dom] / (seg_ms[dom] * 1e-3) / 1e9, "peak": NVLINK_GBS,
                "unit": "GB/s", "traffic": None, "algorithmic_bytes": link[dom],
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "traffic": None, "algorithmic_bytes": alg[dom],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "peak_kind": "copy (1:1 read/write); the combine gather reads K rows per row it "
                             "writes, and read-dominated traffic can exceed the copy rate"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # DRAM bytes per launch of the same kernel from the committed ncu --set
    # full capture of this command (profiles/ncu_traffic.json, qwen3 at N=1)
    tr_path = ROOT / "profiles" / "ncu_traffic.json"
    if (roof["bound"] == "hbm" and world == 1 and args.config == "qwen3" and args.tokens is None
            and tr_path.exists()):
        tr = json.loads(tr_path.read_text())["dram_bytes_per_launch"]
        names = {"pack": ("k_pack_local", "k_pack")}.get(dom, ("k_" + dom,))
        roof["traffic"] = next((tr[n] for n in names if n in tr), None)
        roof["traffic_source"] = "profiles/ncu_traffic.json (ncu --set full, dram read+write)"
    per_kernel = {k: {"ms": round(seg_ms[k], 4), "bytes": alg[k],
                      "GBps": round(alg[k] / max(seg_ms[k], 1e-9) / 1e6, 1)} for k in alg}
    for k in link:
        per_kernel[k]["link_GBps"] = round(link[k] / max(seg_ms[k], 1e-9) / 1e6, 1)
    tokens_total = G * T_r
    value = tokens_total / (ms * 1e-3)

    # end-to-end through the public API with host buffers (pinned), copies timed:
    # every step copies its inputs host -> device, routes, dispatches, combines
    # and copies the output back.  Double-buffered across steps: step i+1's H2D
    # (copy-in stream) and step i-1's D2H (copy-out stream) overlap step i's
    # kernels, so the step rate is bounded by the PCIe direction that moves more.
    e2e = None
    if not args.no_e2e:
        # pinned host buffers on the GPU's own NUMA node: bind this process to
        # the CPUs NVML reports as local to the GPU before allocating (first
        # touch places the pages), so the copies do not cross the socket link
        numa_cpus, old_aff = _bind_gpu_local_cpus(local)
        hx = [torch.empty(T, M, dtype=dtype).pin_memory() for _ in range(2)]
        hl = [torch.empty(T, E, dtype=torch.float32).pin_memory() for _ in range(2)]
        for b in range(2):
            hx[b].copy_(x.cpu())
            hl[b].copy_(logits.cpu())
        ho = [torch.empty(T, M, dtype=dtype).pin_memory() for _ in range(2)]
        for b in range(2):
            ho[b].zero_()        # first touch on the bound CPUs
        if old_aff:
            os.sched_setaffinity(0, old_aff)
        dx = [torch.empty_like(x) for _ in range(2)]
        dl = [torch.empty_like(logits) for _ in range(2)]
        do = [torch.empty_like(out) for _ in range(2)]
        comp = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        h2d_done = [ev(), ev()]
        comp_done = [ev(), ev()]
        d2h_done = [ev(), ev()]
        for b in range(2):   # all buffers start free
            comp_done[b].record(comp)
            d2h_done[b].record(comp)

        def e2e_step(i):
            b = i % 2
            with torch.cuda.stream(s_in):
                s_in.wait_event(comp_done[b])          # step i-2 finished reading dx[b]
                dx[b].copy_(hx[b], non_blocking=True)
                dl[b].copy_(hl[b], non_blocking=True)
                h2d_done[b].record(s_in)
            comp.wait_event(h2d_done[b])
            comp.wait_event(d2h_done[b])               # out[b] of step i-2 copied out
            slot, wts, _ = route_topk(dl[b], K)
            ep.dispatch(dx[b], slot, wts, dedup=MODE)
            ep.combine(slot, wts, dedup=MODE, out=do[b])
            comp_done[b].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[b])
                ho[b].copy_(do[b], non_blocking=True)
                d2h_done[b].record(s_out)

        step(ep, MODE, out)   # device-resident reference output for the check below
        for i in range(4):
            e2e_step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_e2e = max(4, args.steps // 2)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(comp)
        s_in.wait_event(s0)
        s_out.wait_event(s0)
        for i in range(n_e2e):
            e2e_step(i)
        comp.wait_event(d2h_done[(n_e2e - 1) % 2])
        comp.wait_event(d2h_done[n_e2e % 2])
        s1.record(comp)
        s1.synchronize()
        t = torch.tensor([s0.elapsed_time(s1) / n_e2e], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        assert torch.equal(ho[(n_e2e - 1) % 2].cuda(), out), "e2e output differs from device run"
        e2e = {"value": tokens_total / (e2e_ms * 1e-3), "unit": "tokens/s",
               "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(hx[0].numel() * 2 + hl[0].numel() * 4),
               "d2h_bytes_per_step": int(ho[0].numel() * 2),
               "pipeline": "double-buffered: H2D(i+1) and D2H(i-1) overlap step i",
               "host_cpus": numa_cpus}

    # config C's two-level dedup over virtual 2x4 GPU groups (HD2: relay to the
    # level-1 group, re-dedup inside it) next to the flat per-GPU dedup, and
    # the reference time model's choice between them under B200 alpha/beta
    hd2 = None
    if args.config == "dsv3" and not args.no_hd2:
        from paper_2508_09591_b200.layer import TwoLevelWorld
        import paper_2508_09591_b200 as hm
        from paper_2508_09591_b200.traffic import _Model
        raw_ep.close()
        all_ep.close()
        tw = TwoLevelWorld((2, 4), E, K, M, T_r, gpus=world, gpu_index=rank,
                           n_cap_rows=2 * T_r * K)

        def step_hd2():
            slot, wts, _ = route_topk(logits, K)
            tw.dispatch(x, slot, wts, dedup2="remote")
            tw.combine(slot, wts, dedup2="remote", out=out)

        for _ in range(max(3, args.warmup)):
            step_hd2()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_h, tot = max(5, args.steps // 4), 0.0
        for _ in range(n_h):
            flush.zero_()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record()
            step_hd2()
            h1.record()
            h1.synchronize()
            tot += h0.elapsed_time(h1)
        th = torch.tensor([tot / n_h], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(th, op=dist.ReduceOp.MAX)
        tw.phase1.check_status()
        tw.phase2.check_status()
        tw.close()
        slot_g, _, _ = route_topk(logits, K)
        topo = hm.build_topology([2, 4], E, M, 2)
        p = PLANNER_CASES[1][4]
        red = (lambda t_: dist.all_reduce(t_)) if world > 1 else None
        mdl = _Model(hm.mask_from_ids(slot_g, E), topo, hm.LevelParams(*p), None, True,
                     red).fetch()
        hd2 = {"topology": [2, 4], "ms_per_step": float(th.item()),
               "vs_flat_per_gpu_dedup": float(th.item()) / ms,
               "d_star_b200_params": int(mdl.d_star),
               "model_times_s": [float(v) for v in mdl.times],
               "note": "d_star_b200_params: the reference time model's choice (traffic.py:"
                       "188-221) with the B200 alpha/beta fits; ms_per_step: d = 2 run as two "
                       "exchanges through relay ranks (TwoLevelWorld).  The layer's per-GPU "
                       "dedup is the d = 2 copy list at GPU level in one exchange plus the "
                       "destination's re-expansion (at N = 2 the level-1 groups are the GPUs)"}

    # full layer forward + backward: gating, dedup dispatch, tcgen05 SwiGLU
    # experts, combine; backward: combine-bwd, tcgen05 FFN bwd, dispatch-bwd
    layer_fwd = None
    if not args.no_layer:
        from paper_2508_09591_b200.moe import HierMoELayer
        inter = INTER[args.config]
        ep.close()
        all_ep.close()
        raw_ep.close()
        if args.config == "dsv3":
            layer_fwd = dsv3_layer_forward(G, E, K, M, inter, T_r, world, rank, x, flush,
                                           tokens_total, max(5, args.steps // 10), peaks)
    if not args.no_layer and args.config != "dsv3":
        layer = HierMoELayer(G, E, K, M, inter, T_r, gpus=world, gpu_index=rank, dedup=MODE,
                             grad=True, n_cap_rows=3 * T_r * K)
        lout = torch.empty(T, M, dtype=dtype, device="cuda")
        gout = torch.randn(T, M, device="cuda", generator=gen).to(dtype)
        for _ in range(3):
            layer(x, out=lout)
            layer.backward(gout)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_l = max(5, args.steps // 10)
        acc = np.zeros(4)
        with ClockSampler(local) as lclk:
            # the public forward / backward (overlaps included: at N > 1 the
            # dispatch moves inside the expert GEMM, the dispatch backward runs
            # beside the weight-gradient GEMMs)
            for _ in range(n_l):
                flush.zero_()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                ev[0].record()
                layer(x, out=lout)
                ev[1].record()
                layer.backward(gout)
                ev[2].record()
                ev[2].synchronize()
                acc += [ev[0].elapsed_time(ev[1]), 0.0, ev[1].elapsed_time(ev[2]),
                        ev[0].elapsed_time(ev[2])]
            # the expert FFN alone (ffn_roofline): serial dispatch, then the GEMMs
            for _ in range(n_l):
                flush.zero_()
                slot_l, w_l, ex_l = layer.route_saved(x)
                layer.world.set_fused(layer.fused_now())
                layer.world.dispatch(x, slot_l, w_l, dedup=layer.dedup)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record()
                layer.experts_forward()
                ev[1].record()
                ev[1].synchronize()
                layer.world.combine(slot_l, w_l, dedup=layer.dedup, out=lout)
                acc[1] += ev[0].elapsed_time(ev[1])
        t = torch.tensor(acc / n_l, dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        fl = layer.flops_per_forward()
        fl_t = torch.tensor([float(fl)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(fl_t, op=dist.ReduceOp.MAX)
        fwd_ms, ffn_ms, bwd_ms, tot_ms = (float(v) for v in t.tolist())
        ffn_tflops = fl_t.item() / (ffn_ms * 1e-3) / 1e12
        # the FFN is timed inside a long loop of layer steps (power-capped
        # clocks): its denominator is the sustained bf16 peak, the burst one
        # (a GEMM timed alone) is reported beside it
        peak_burst = peaks.get("bf16_tflops", 1590.0)
        peak_tf = peaks.get("bf16_tflops_sustained", peak_burst)
        layer_fwd = {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "fwd_bwd_ms": tot_ms,
                     "fwd_tokens_per_s": tokens_total / (fwd_ms * 1e-3),
                     "fwd_bwd_tokens_per_s": tokens_total / (tot_ms * 1e-3),
                     "ffn_fwd_ms": ffn_ms, "ffn_flops_per_gpu": int(fl_t.item()),
                     "ffn_roofline": {"bound": "tensor", "achieved": ffn_tflops, "peak": peak_tf,
                                      "unit": "TFLOP/s", "frac": ffn_tflops / peak_tf,
                                      "peak_kind": "sustained" if peak_tf != peak_burst
                                      else "burst",
                                      "peak_burst": peak_burst,
                                      "frac_burst": ffn_tflops / peak_burst,
                                      "kernel": "k_grouped_gemm_pair (tcgen05, 2 GEMMs, fwd)"},
                     "inter": inter, "transport": layer.dedup, "clocks": lclk.summary(),
                     "note": "router GEMMs, gate backward, dispatch/combine and experts fwd+bwd "
                             "are our kernels"}
        layer.close()

    planner = None
    if world == 1 and not args.no_planner:
        planner = planner_gpu(G * T_r, K)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(args.config, 5, 1, args.tokens)
        if planner is not None:
            cpu_pl = planner_cpu(G * T_r, K)
            for name in planner:
                planner[name]["cpu_ms"] = cpu_pl[name]
            planner["cpu_cores"] = os.cpu_count()

    if nccl is not None and link_dedup:
        # communication alone: NCCL's two row AlltoAlls vs our dedup pushes
        # (pack + pre-reduced return), both device-timed
        nccl["comm_speedup_dedup_vs_nccl"] = nccl["exchange_ms"] / link_dedup
        nccl["dedup_link_ms"] = link_dedup
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "us_per_layer": ms * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": desc, "ranks": G, "gpus": world, "ranks_per_gpu": L,
                       "experts": E, "top_k": K, "hidden": M, "tokens_per_rank": T_r,
                       "global_tokens": tokens_total, "dedup_level": "GPU (EP rank)",
                       "l2": "256 MB buffer written between timed steps (> 126 MB L2)",
                       "timed": "route+plan+notify+pack+expand | reduce+gather (+barriers)"},
            "dispatch_us": 1e3 * (seg_ms["plan"] + seg_ms["notify"] + seg_ms["pack"]
                                  + seg_ms["barrier1"] + seg_ms["expand"]),
            "combine_us": 1e3 * (seg_ms["reduce"] + seg_ms["barrier2"] + seg_ms["gather"]),
            "kernel_ms": {k: round(v, 4) for k, v in seg_ms.items()},
            "kernels": per_kernel,
            "dispatch": "fused: row indices (local tokens / received rows), GEMM1 gathers the "
                        "rows with cp.async producer warps" if FUSED
                        else "copy: rows to the expert-major buffers",
            "materialized_dispatch": None if not FUSED else {
                "ms_per_step": ms_copy, "value": tokens_total / (ms_copy * 1e-3),
                "kernel_ms": {k: round(v, 4) for k, v in zip(SEGMENTS, seg_copy.tolist())},
                "note": "the same step with the expert-major rows materialised (copying pack "
                        "and destination re-expansion)"},
            "transport": MODE,
            "transport_choice": {"mode": choice.mode, "d_star": choice.d_star,
                                 "times_s": list(choice.times),
                                 "time_without_dedup_s": choice.time_without_dedup,
                                 "runtime_topology": list(rtopo.level_fanouts),
                                 "rule": "reference pick_dimension over dedup times; no dedup "
                                         "only if strictly faster (transport.py)"},
            "nodedup": {"ms_per_step": ms_raw, "value": tokens_total / (ms_raw * 1e-3),
                        "kernel_ms": {k: round(v, 4) for k, v in zip(SEGMENTS, seg_raw.tolist())},
                        "speedup_dedup_vs_nodedup": ms_raw / ms,
                        "link_time_ratio": link_raw / max(link_dedup, 1e-9) if link_dedup else None},
            "nccl_nodedup": nccl,
            "cuda_graph_ms_per_step": graph_ms,
            "hd2_2x4": hd2,
            "dedup_all_ranks": {"ms_per_step": ms_all,
                                "kernel_ms": {k: round(v, 4) for k, v in zip(SEGMENTS, seg_all.tolist())}},
            "comm_bytes": {"dedup_rows_out": rows_dedup_out, "raw_rows_out": rows_raw_out,
                           "dedup_remote_bytes": rem_dedup * rb, "raw_remote_bytes": rem_raw * rb,
                           "rank_dedup_remote_bytes": rem_rank_dedup * rb,
                           "row_ratio_raw_over_dedup": rows_raw_out / max(1, rows_dedup_out),
                           "remote_byte_ratio_raw_over_dedup":
                               (rem_raw / rem_dedup) if rem_dedup else None},
            "roofline": roof,
            "link_roofline": None if world == 1 else {
                "bound": "nvlink", "kernel": "dispatch+combine pushes",
                "achieved": (link["pack"] + link[ret_key]) / (link_dedup * 1e-3) / 1e9,
                "peak": NVLINK_GBS, "unit": "GB/s",
                "frac": (link["pack"] + link[ret_key]) / (link_dedup * 1e-3) / 1e9 / NVLINK_GBS,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction",
                "sm_push_ceiling": SM_PUSH_GBS,
                "frac_of_sm_push_ceiling":
                    (link["pack"] + link[ret_key]) / (link_dedup * 1e-3) / 1e9 / SM_PUSH_GBS,
                "sm_push_source": "tools/link_probe.cu all-to-all SM pushes (16-B stores / TMA "
                                  "bulk), profiles/r01_link_probe.jsonl"},
            "cpu_baseline": None if cpu is None else
            {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": e2e,
            "layer_fwd": layer_fwd,
            "planner": planner,
            "gpu_launches": main_launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), file=out_stream, flush=True)
    ep.close()
    raw_ep.close()
    all_ep.close()  # (closing twice is a no-op)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

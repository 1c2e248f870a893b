"""Benchmark of the PP stage-boundary transfer under 1F1B (BASELINE.json metric:
"stage-boundary P2P GB/s vs NVLink; 1F1B tokens/s device-direct vs CPU-fwd").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ppc|reference]

Workload (BASELINE.json configs[1], "C2"): LLaMA-8B-shaped boundary [1,4096,4096] bf16
(32 MiB per message), PP = 2, M = 8 micro-batches, non-interleaved 1F1B, comm-only step
(identity stage functions, R13).  A step = every FWD and BWD send/recv of one
1F1B step of every pipeline.
  * N = 1: the two stages are virtual stages on one GPU (the intra-device ring, K11);
  * N >= 2: one process per GPU (torchrun), N/2 independent PP=2 pipelines (weak scaling,
    no data-path collective), rings mapped over NVLink with CUDA IPC.
value = tokens/s of the whole job = pipelines * M * seq * K / T, T = max over ranks of the
CUDA-event time of the K timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1F1B tokens/s (stage-boundary P2P, device-direct)"
NVLINK_GBPS = 900.0          # NVLink 5 per direction per GPU (nominal; R4)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ppc", choices=["ppc", "reference"])
    ap.add_argument("--pp", type=int, default=2)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--engine", default="sm", choices=["sm", "ce", "pull"])
    ap.add_argument("--chunk", type=int, default=0,
                    help="flag / pull granularity; 0 = tuned default (256 KiB zero-copy, "
                         "512 KiB ring push, 128 KiB virtual stages)")
    ap.add_argument("--channels", type=int, default=1)
    ap.add_argument("--cta", type=int, default=0)
    ap.add_argument("--slots", type=int, default=0, help="ring slots K; 0 = pp + 1")
    ap.add_argument("--graph", type=int, default=1,
                    help="replay the step as one CUDA graph (ppc_graph_create)")
    ap.add_argument("--zc", type=int, default=-1,
                    help="N>=2: register the step's source buffers (zero-copy NVLink pulls); "
                         "-1 = on for pp = 2 (every send is then a pull), off for deeper "
                         "pipelines: a pull moves data only when the receiver reaches its "
                         "receive, while a push runs ahead into the K-slot ring, which the "
                         "warm-up of a deep 1F1B pipeline exploits (PP4 M16: 3623 us "
                         "all-pull vs 2868 us, profiles/r38_pp4_zc_vs_ring.jsonl)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks (NVML, during timing)
class ClockSampler:
    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:          # NVML missing: report nulls
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.001)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def ncu_traffic(key):
    """Per-launch dram read+write bytes of the dominant kernel from a committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


def pcie_roofline(world, h2d_gpu, d2h_gpu, ms_step):
    """The e2e step's host-link bound: each GPU's H2D and D2H bytes at the pinned-copy rates
    measured with both directions busy and `world` GPUs copying at once
    (profiles/pcie_roofline.json); null when that GPU count was not measured."""
    try:
        with open(os.path.join(ROOT, "profiles", "pcie_roofline.json")) as fh:
            r = json.load(fh)["both_dirs_gbps"].get(str(world))
    except Exception:
        r = None
    if not r:
        return None
    bound_ms = max(h2d_gpu / (r["h2d"] * 1e6), d2h_gpu / (r["d2h"] * 1e6))
    return {"bound": "pcie+host", "bound_ms_per_step": bound_ms, "frac": bound_ms / ms_step,
            "h2d_gbps": r["h2d"], "d2h_gbps": r["d2h"],
            "source": "profiles/pcie_roofline.json (tools/nvlink_probe pcie, r58)"}


# ---------------------------------------------------------------- CPU oracle legs
def oracle_step_sample(M_sample, nbytes, seed=42):
    """One bounded sample of the workload on the CPU oracle: a PP=2 1F1B step over M_sample
    micro-batches of the same boundary tensors (identity stages), byte-level transfers with
    header checks and digests (oracle/proxy.py + oracle/transfer.py).  Returns seconds."""
    import numpy as np
    from oracle.proxy import run_1f1b
    from synth import payload as P
    t0 = time.perf_counter()
    X = {m: P.source_activation(seed, 0, m, nbytes) for m in range(M_sample)}
    G = {m: P.source_gradient(seed, 0, m, nbytes) for m in range(M_sample)}
    ident = lambda s, m, x: x
    Y, DX, chans, _ = run_1f1b(2, M_sample, 2, ident, ident, X.__getitem__, G.__getitem__,
                               nbytes, nbytes, nbytes)
    assert all(np.array_equal(Y[m], X[m]) for m in range(M_sample))
    return time.perf_counter() - t0


def cpu_baseline(args, nbytes):
    M_s = 2
    secs = oracle_step_sample(M_s, nbytes)
    reps = max(1, min(5, int(15.0 / max(secs, 1e-3))))
    times = [secs] + [oracle_step_sample(M_s, nbytes) for _ in range(reps - 1)]
    t = statistics.median(times)
    return {"value": M_s * args.seq / t, "unit": "tokens/s", "cores": 1, "kind": "oracle",
            "sample": f"PP=2 1F1B step over {M_s} of the {args.M} micro-batches "
                      f"([1,{args.seq},{args.hidden}] bf16 = {nbytes} B messages), "
                      f"byte-level ring transfer with header checks + blake2b digests, "
                      f"median of {len(times)} runs, single thread"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nbytes = args.seq * args.hidden * 2
    M_s = 2
    for _ in range(args.warmup):
        oracle_step_sample(M_s, nbytes)
    t = sum(oracle_step_sample(M_s, nbytes) for _ in range(args.steps))
    value = M_s * args.seq * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": workload_config(args, pipelines=1, virtual=False),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                             "sample": f"PP=2 1F1B step over {M_s} micro-batches per step"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, pipelines, virtual):
    name = "C2: " if (args.pp, args.hidden, args.M) == (2, 4096, 8) else ""
    model = "Qwen2-7B" if args.hidden == 3584 else "LLaMA-8B"
    return {"workload": f"{name}{model}-shaped PP={args.pp} boundary [1,{args.seq},{args.hidden}] "
                        f"bf16, M={args.M}, 1F1B comm-only step",
            "pp": args.pp, "pipelines": pipelines, "virtual_stages": virtual, "M": args.M,
            "seq": args.seq, "hidden": args.hidden, "msg_bytes": args.seq * args.hidden * 2,
            "engine": args.engine, "chunk_bytes": args.chunk, "channels": args.channels,
            "ring_slots": args.slots or args.pp + 1, "zero_copy_sends": bool(args.zc) and not virtual,
            "cuda_graph": bool(args.graph),
            "l2": l2_note(args)}


def l2_note(args):
    """How the timing rule on L2 is met: the per-stage working set of one step vs 126 MB L2."""
    msg = args.seq * args.hidden * 2
    per_dir = args.M * msg
    if per_dir > 126 * 10**6:
        return (f"inputs larger than L2 (M x {msg / 2**20:g} MiB per stage per direction, "
                f"{per_dir / 2**20:g} MiB)")
    return f"inputs fit in L2 ({per_dir} B per stage per direction): latency run, not a bench line"


# ---------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_2602_18007_b200 as ppc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    distributed = world > 1
    if distributed:
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    if args.zc < 0:
        args.zc = 1 if args.pp == 2 else 0
    if args.engine == "ce":
        args.graph = 0        # the CE engine's host-resolved slots are not graph-capturable
    if not args.chunk:
        # tuned on 2x B200 (profiles/r1_tune_step_ws.jsonl): 512 KiB chunks x 64 CTAs
        # zero-copy pulls: 256 KiB grain; ring push: 512 KiB (profiles/r11_tune_zero_copy.jsonl)
        args.chunk = ((256 if args.zc else 512) << 10) if distributed else (128 << 10)
    S = args.pp
    nbytes = args.seq * args.hidden * 2
    M = args.M
    engine = {"sm": ppc.ENGINE_SM, "ce": ppc.ENGINE_CE, "pull": ppc.ENGINE_PULL}[args.engine]
    cfg = ppc.make_config(tp=1, pp=S, dp=max(1, world // S) if distributed else 1,
                          max_msg_bytes=nbytes, ring_slots=args.slots, channels=args.channels,
                          chunk_bytes=args.chunk, engine=engine, cta_per_channel=args.cta,
                          trace=3)
    if distributed:
        if world % S:
            raise SystemExit(f"--gpus {world} is not a multiple of pp={S}")
        comms = [ppc.connect_distributed(cfg, rank, world, local, with_nccl=False)]
        stages = [comms[0].group(ppc.GROUP_PP)[0].index(rank)]
        pipelines = world // S
    else:
        comms = ppc.virtual_stages(cfg, dev)
        stages = list(range(S))
        pipelines = 1

    def bufs():
        return [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(M)]

    X = {s: bufs() for s in stages if s == 0}
    G = {s: bufs() for s in stages if s == S - 1}
    Y = {s: bufs() for s in stages if s == S - 1}
    DX = {s: bufs() for s in stages if s == 0}
    for s in stages:
        for m in range(M):
            if s in X:
                ppc.fill_payload(X[s][m], nbytes, 42, 0, 0xFF, 0, m)
            if s in G:
                ppc.fill_payload(G[s][m], nbytes, 42, 0, 0xFF, 1, m)
    args_dev = [ppc.StepArgs(M, nbytes, nbytes, x=X.get(s), g=G.get(s), y=Y.get(s),
                             dx=DX.get(s)) for s in stages]
    streams = [torch.cuda.Stream() for _ in stages]
    if distributed and args.zc:
        # zero-copy: the stage inputs X / G are registered send buffers; receivers pull them
        ppc.register_tensors(comms[0], [t for s in stages for t in X.get(s, []) + G.get(s, [])])

    graph = [None]

    def one_step(a=None, eager=False):
        if graph[0] is not None and a is None and not eager:
            graph[0].launch()
            return
        a = a or args_dev
        if distributed:
            ppc.step_1f1b(comms[0], a[0], streams[0])
        else:
            ppc.step_1f1b_local(comms, a, streams)

    def barrier():
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()

    def max_over_ranks(v):
        if not distributed:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    one_step(eager=True)                 # allocates the step buffers
    barrier()
    if args.graph:                       # the whole step as one CUDA graph per process
        graph[0] = ppc.StepGraph(comms, args_dev, streams)
    for _ in range(args.warmup):
        one_step()
    barrier()

    def timed_region(instrumented: bool):
        """K steps between barriers + synchronize; CUDA events on every stage stream (the
        launch stream for graph replays); max over ranks.  instrumented: eager steps with
        CUDA-event pairs around every transfer launch."""
        for c in comms:
            c.set_trace(2 if instrumented else 0)
            c.kernel_times(0), c.kernel_times(1)
        sts = streams[:1] if (graph[0] is not None and not instrumented) else streams
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in sts]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in sts]
        barrier()
        for e, st in zip(ev0, sts):
            e.record(st)
        for _ in range(args.steps):
            one_step(eager=instrumented)
        for e, st in zip(ev1, sts):
            e.record(st)
        barrier()
        return max_over_ranks(max(a.elapsed_time(b) for a, b in zip(ev0, ev1)))

    # ---- headline timed region (no instrumentation), clocks sampled during it
    sampler = ClockSampler(dev)
    sampler.start()
    ms_total = timed_region(False)
    clocks = sampler.stop()
    ms_step = ms_total / args.steps
    tokens = pipelines * M * args.seq * args.steps
    value = tokens / (ms_total * 1e-3)
    # ---- the same K steps again with per-launch CUDA events for the kernel roofline
    n_rec0 = [len(c.trace()) for c in comms]
    ms_instr = timed_region(True)
    push_ms = [t for c in comms for t in c.kernel_times(0)]
    recv_ms = [t for c in comms for t in c.kernel_times(1)]
    # device-side %globaltimer records of the receives of that pass: a zero-copy receive's
    # record starts when the publication is seen, so t_end - t_start is its pull (data phase)
    recv_recs = [r for c, n0 in zip(comms, n_rec0) for r in c.trace()[n0:] if r["kind"] == 1]
    for c in comms:
        c.set_trace(0)
    n_launch_local = len(push_ms) + len(recv_ms)
    n_launch = n_launch_local
    if distributed:
        t = torch.tensor([n_launch_local], dtype=torch.float64)
        dist.all_reduce(t)
        n_launch = int(t.item())

    # dominant kernel: the one that moves the bytes — N=1: the hand-off copy; N>=2 zero-copy:
    # the receiver's NVLink pull (recv_kernel; its launch also spans the wait for the peer's
    # publication); N>=2 ring: the SM push
    zc_dom = distributed and bool(args.zc)
    dom_ms = recv_ms if zc_dom else push_ms
    avg_push_ms = statistics.mean(dom_ms) if dom_ms else float("nan")
    avg_push_ms = max_over_ranks(avg_push_ms)
    peaks = measured_peaks()
    if distributed:
        alg = nbytes                                  # bytes that cross NVLink per launch
        peak, unit, bound = NVLINK_GBPS, "GB/s", "nvlink"
        peak_src = "NVLink 5 nominal 900 GB/s per direction (guide measured peer copy 770)"
    else:
        alg = 2 * nbytes                              # HBM read + write per launch
        peak = peaks.get("hbm_gbs", 6650.0)
        unit, bound = "GB/s", "hbm"
        peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    achieved = alg / (avg_push_ms * 1e-3) / 1e9
    if not distributed:
        if os.environ.get("PPC_COPY_TMA_CTAS", "0") != "0":
            kname, tkey = "ppc::copy_tma_kernel (virtual-stage TMA bulk hand-off)", "copy_tma_n1"
        else:
            kname, tkey = "ppc::copy_kernel (virtual-stage SIMT hand-off)", "copy_n1"
    elif zc_dom:
        kname = ("ppc::recv_kernel (zero-copy NVLink pull into the user buffer; CUDA events "
                 "on its stream, so the launch time includes the wait for the publication)")
        tkey = "recv_n2"
    else:
        kname, tkey = "ppc::push_ws_kernel (SM push over NVLink)", "push_n2"
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": ncu_traffic(tkey),
            "kernel": kname, "alg_bytes_per_launch": alg,
            "avg_launch_us": avg_push_ms * 1e3, "launches_timed": len(dom_ms),
            "peak_source": peak_src,
            "timed_region": "second pass of the same K steps with per-launch CUDA events "
                            f"(step {ms_instr / args.steps:.3f} ms instrumented vs {ms_step:.3f} plain)",
            "step_aggregate": {"bytes_per_step": alg * len(dom_ms) / max(1, args.steps),
                               "achieved": alg * len(dom_ms) / (ms_instr * 1e-3) / 1e9,
                               "achieved_plain": alg * len(dom_ms) / max(1, args.steps)
                                                 / (ms_step * 1e-3) / 1e9,
                               "frac_plain": alg * len(dom_ms) / max(1, args.steps)
                                             / (ms_step * 1e-3) / 1e9 / peak,
                               "note": "this process's transfer launches of the step (both "
                                       "directions, concurrent) over the instrumented step "
                                       "time (achieved) and over the un-instrumented headline "
                                       "step time (achieved_plain)"},
            "send_avg_launch_us": (statistics.mean(push_ms) * 1e3) if push_ms else None,
            "recv_avg_launch_us": (statistics.mean(recv_ms) * 1e3) if recv_ms else None}
    # launches of the dominant kernel overlap (the F and B transfers of a 1F1B step run
    # concurrently and share the bandwidth), so per-launch "achieved" is ~1/concurrency of
    # what the kernel class moves; report the measured overlap beside it
    if dom_ms and ms_instr > 0:
        conc = sum(dom_ms) / ms_instr        # this process's launches (all its stages)
        roof["concurrency"] = conc
        roof["frac_x_concurrency"] = roof["frac"] * conc
    if distributed and args.zc and recv_recs:
        phase_us = statistics.mean((r["t_end_ns"] - r["t_start_ns"]) * 1e-3 for r in recv_recs)
        phase_us = max_over_ranks(phase_us)
        roof["zero_copy_pull_data_phase"] = {
            "avg_us": phase_us, "achieved": nbytes / (phase_us * 1e-6) / 1e9, "unit": "GB/s",
            "frac": nbytes / (phase_us * 1e-6) / 1e9 / peak, "records": len(recv_recs),
            "timing": "%globaltimer stamps in recv_kernel: publication seen -> last CTA done"}
    boundary_gbps = 2 * M * nbytes * pipelines * (S - 1) * args.steps / (ms_total * 1e-3) / 1e9

    # ---- e2e: the same step through the C-ABI with pinned HOST inputs / outputs
    e2e = None
    if not args.no_e2e:
        def hbufs():
            return [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(M)]
        hX = {s: hbufs() for s in X}
        hG = {s: hbufs() for s in G}
        hY = {s: hbufs() for s in Y}
        hDX = {s: hbufs() for s in DX}
        for s in hX:
            for m in range(M):
                hX[s][m].copy_(X[s][m].cpu())
        for s in hG:
            for m in range(M):
                hG[s][m].copy_(G[s][m].cpu())
        args_host = [ppc.StepArgs(M, nbytes, nbytes, x=hX.get(s), g=hG.get(s), y=hY.get(s),
                                  dx=hDX.get(s)) for s in stages]
        K2 = max(3, min(args.steps, 10))
        one_step(args_host)
        barrier()
        e0 = [torch.cuda.Event(enable_timing=True) for _ in stages]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in stages]
        for e, st in zip(e0, streams):
            e.record(st)
        for _ in range(K2):
            one_step(args_host)
        for e, st in zip(e1, streams):
            e.record(st)
        barrier()
        ms_e2e = max_over_ranks(max(a.elapsed_time(b) for a, b in zip(e0, e1)))
        h2d = (len(hX) + len(hG)) * M * nbytes
        d2h = (len(hY) + len(hDX)) * M * nbytes
        if distributed:
            t = torch.tensor([h2d, d2h], dtype=torch.float64)
            dist.all_reduce(t)
            h2d, d2h = int(t[0]), int(t[1])
        ok = all(torch.equal(hY[s][m], X[0][m].cpu()) for s in hY for m in (0, M - 1)) \
            if (hY and 0 in X) else None
        e2e = {"value": pipelines * M * args.seq * K2 / (ms_e2e * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ms_e2e / K2, "steps": K2, "outputs_checked": ok,
               "roofline": pcie_roofline(world, h2d / world, d2h / world, ms_e2e / K2)}
        for c in comms:
            c.kernel_times(0), c.kernel_times(1)

    cpu = None
    if rank == 0 and not distributed and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, nbytes)

    bad = [c.poll() for c in comms if c.poll() != 0]
    if rank == 0:
        msg_us = nbytes / (NVLINK_GBPS * 1e3)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": workload_config(args, pipelines, not distributed),
            "boundary_gbps": boundary_gbps,
            "step_roofline_us_pp2": (M + 1) * msg_us if S == 2 else None,
            "frac_of_step_roofline": ((M + 1) * msg_us / (ms_step * 1e3)) if S == 2 else None,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": n_launch, "errors": [ppc.STATUS[b] for b in bad],
        }
        print(json.dumps(line), flush=True)
    barrier()
    if graph[0] is not None:
        graph[0].destroy()
    for c in comms:
        c.disconnect()
    if distributed:
        dist.barrier()
    for c in comms:
        c.destroy()
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

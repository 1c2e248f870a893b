"""Benchmark of the PP stage-boundary transfer under 1F1B (BASELINE.json metric:
"stage-boundary P2P GB/s vs NVLink; 1F1B tokens/s device-direct vs CPU-fwd").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ppc|reference]

Headline workload (BASELINE.json configs[1], "C2"): LLaMA-8B-shaped boundary [1,4096,4096]
bf16 (32 MiB per message), PP = 2, M = 8 micro-batches, non-interleaved 1F1B, comm-only step
(identity stage functions, R13).  A step = every FWD and BWD send/recv of one 1F1B
step of every pipeline.
  * N = 1: the two stages are virtual stages on one GPU: the single-copy hand-off (headline)
    and, beside it, the intra-device ring (push into the ring slot + copy-out);
  * N >= 2: one process per GPU (torchrun), N/2 independent PP=2 pipelines (weak scaling,
    no data-path collective), rings and registered buffers mapped over NVLink (CUDA IPC).
value = tokens/s of the whole job = pipelines * M * seq * K / T, T = max over ranks of the
CUDA-event time of the K timed steps.  Beside the headline, the same run measures: the
BASELINE north-star configurations that fit the GPU count (N = 4: PP4 M16 (C3 per TP
pipeline) and PP4 M32 Qwen (C4 stand-in); N = 8: C3 = PP4 x TP2 M16 with DCBS (NCCL TP
groups) and C4 = PP8 M32 Qwen), the CPU-Forwarding baseline B1 (libppcb) on the same
workload, the end-to-end path with host buffers, and the CPU oracle.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1F1B tokens/s (stage-boundary P2P, device-direct)"
NVLINK_GBPS = 900.0          # NVLink 5 per direction per GPU (nominal; R4)

# BASELINE.json configs (SURVEY §8 sizes): name -> (pp, tp, M, hidden, model)
WORKLOADS = {
    "C2": (2, 1, 8, 4096, "LLaMA-8B"),
    "C3": (4, 2, 16, 4096, "LLaMA-8B"),
    "C4": (8, 1, 32, 3584, "Qwen2-7B"),
    "C3-pp4": (4, 1, 16, 4096, "LLaMA-8B"),      # one TP pipeline of C3 (4-GPU stand-in)
    "C4-pp4": (4, 1, 32, 3584, "Qwen2-7B"),      # C4 on 4 GPUs (stand-in)
}
EXTRA = {1: [], 2: [], 4: ["C3-pp4", "C4-pp4"], 8: ["C3", "C4"]}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ppc", choices=["ppc", "reference"])
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--seq", type=int, default=4096)
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
                         "pipelines (a push runs ahead into the K-slot ring, which the warm-up "
                         "of a deep 1F1B pipeline exploits; profiles/r38_pp4_zc_vs_ring.jsonl)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-b1", action="store_true", help="skip the CPU-Forwarding B1 arm")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the north-star configurations beside the headline")
    ap.add_argument("--no-ring", action="store_true", help="N=1: skip the intra-device ring line")
    return ap.parse_args(argv)


# ---------------------------------------------------------------- workload resolution
def resolve(args, world, name=None):
    """The configuration one run of `name` uses at `world` ranks (both arms print it)."""
    name = name or args.workload
    pp, tp, M, hidden, model = WORKLOADS[name]
    virtual = world == 1
    if virtual and (pp != 2 or tp != 1):
        raise SystemExit(f"{name} needs {pp * tp} GPUs")
    if not virtual and world % (pp * tp):
        raise SystemExit(f"--gpus {world} is not a multiple of pp*tp = {pp * tp}")
    zc = args.zc if args.zc >= 0 else (1 if pp == 2 else 0)
    zc = bool(zc) and not virtual
    chunk = args.chunk or ((128 << 10) if virtual else ((256 << 10) if zc else (512 << 10)))
    pipelines = 1 if virtual else world // pp
    return {"name": name, "pp": pp, "tp": tp, "dp": 1 if virtual else world // (pp * tp),
            "M": M, "seq": args.seq, "hidden": hidden, "model": model,
            "msg_bytes": args.seq * hidden * 2, "virtual": virtual, "pipelines": pipelines,
            "zc": zc, "chunk": chunk, "engine": args.engine, "channels": args.channels,
            "cta": args.cta, "slots": args.slots or pp + 1,
            "graph": bool(args.graph) and args.engine != "ce"}


def config_dict(wl, world):
    tag = f"{wl['name']}: " if wl["name"] in ("C2", "C3", "C4") else f"{wl['name']} (stand-in): "
    layout = (f"PP={wl['pp']} x TP={wl['tp']} (DCBS: NCCL TP groups, custom-kernel PP)"
              if wl["tp"] > 1 else f"PP={wl['pp']}")
    where = ("two virtual stages on one GPU" if wl["virtual"] else
             f"{wl['pipelines']} independent pipeline(s) on {world} GPUs")
    per_dir = wl["M"] * wl["msg_bytes"]
    return {"workload": f"{tag}{wl['model']}-shaped {layout} boundary [1,{wl['seq']},"
                        f"{wl['hidden']}] bf16, M={wl['M']}, 1F1B comm-only step, {where}",
            "pp": wl["pp"], "tp": wl["tp"], "pipelines": wl["pipelines"],
            "virtual_stages": wl["virtual"], "M": wl["M"], "seq": wl["seq"],
            "hidden": wl["hidden"], "msg_bytes": wl["msg_bytes"], "engine": wl["engine"],
            "chunk_bytes": wl["chunk"], "channels": wl["channels"], "ring_slots": wl["slots"],
            "zero_copy_sends": wl["zc"], "cuda_graph": wl["graph"],
            # N=1 hands boundaries over in HBM (two virtual stages), N>=2 over NVLink: the
            # weak-scaling series is N = 2, 4, 8 (same per-pipeline work on the same link)
            "transport": "hbm (intra-device)" if wl["virtual"] else "nvlink (peer pulls)",
            "l2": (f"inputs larger than L2 (M x {wl['msg_bytes'] / 2**20:g} MiB per stage per "
                   f"direction = {per_dir / 2**20:g} MiB > 126 MB)" if per_dir > 126e6 else
                   "inputs fit in L2: latency run, not a bench line")}


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
        while True:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            if self._stop.is_set():
                break
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
    """Per-launch traffic of the dominant kernel from a committed ncu capture
    (profiles/ncu_traffic.json): local DRAM read+write bytes (N = 1) or NVLink bytes (N >= 2)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


def pcie_roofline(world, h2d_gpu, d2h_gpu, ms_step):
    """The e2e step's host-link bound (profiles/pcie_roofline.json); null if unmeasured."""
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
def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or None


def oracle_step(pp, M, nbytes, seed=42):
    """One full 1F1B step of the workload on the CPU oracle (oracle/proxy.py + transfer.py):
    PP stages, M micro-batches of `nbytes` messages each way, byte-level ring transfers with
    header checks and digests, identity stages; outputs checked.  Returns seconds."""
    import numpy as np
    from oracle.proxy import run_1f1b
    from synth import payload as P
    t0 = time.perf_counter()
    X = {m: P.source_activation(seed, 0, m, nbytes) for m in range(M)}
    G = {m: P.source_gradient(seed, 0, m, nbytes) for m in range(M)}
    ident = lambda s, m, x: x
    Y, DX, _, _ = run_1f1b(pp, M, pp + 1, ident, ident, X.__getitem__, G.__getitem__,
                           nbytes, nbytes, nbytes)
    assert all(np.array_equal(Y[m], X[m]) and np.array_equal(DX[m], G[m]) for m in range(M))
    return time.perf_counter() - t0


def _oracle_worker(a):
    return oracle_step(*a)


def cpu_baseline(wl, budget_s=30.0):
    """the oracle as it stands on this host's cores — one full step of the
    headline workload single-process, then P concurrent full steps (one per process, P =
    usable cores bounded by memory) for the all-core throughput."""
    pp, M, nb = wl["pp"], wl["M"], wl["msg_bytes"]
    tokens = wl["M"] * wl["seq"]
    t1 = oracle_step(pp, M, nb)
    cores = len(os.sched_getaffinity(0))
    per_proc = 6 * M * nb                      # X, G, rings, outputs, digests (generous)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    P = max(1, min(cores, int(0.5 * avail // per_proc)))
    tall = None
    if P > 1 and t1 * 1.5 < budget_s:
        ctx = mp.get_context("fork")
        t0 = time.perf_counter()
        with ctx.Pool(P) as pool:
            pool.map(_oracle_worker, [(pp, M, nb)] * P)
        tall = time.perf_counter() - t0
    moved = 2 * (pp - 1) * M * nb             # bytes the step transfers (both directions)
    out = {"value": tokens / t1, "unit": "tokens/s", "cores": 1, "kind": "oracle",
           "sample": f"one full {wl['name']} step (PP={pp}, M={M}, {2 * (pp - 1) * M} messages "
                     f"of {nb} B, byte-level ring transfers + header checks + digests), "
                     f"single process",
           "gib_per_s": moved / t1 / 2**30, "s_per_step": t1, "cpu_model": cpu_model(),
           "host_cores": cores}
    if tall is not None:
        out["all_cores"] = {"value": P * tokens / tall, "unit": "tokens/s", "cores": P,
                            "processes": P, "s_wall": tall,
                            "gib_per_s": P * moved / tall / 2**30,
                            "sample": f"{P} concurrent full steps, one per process"}
    return out


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only), timed on the
    GPU arm's config: every step is one full oracle step of the headline workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = args.gpus
    wl = resolve(args, world)
    tokens = wl["pipelines"] * wl["M"] * wl["seq"]
    pp, M, nb = wl["pp"], wl["M"], wl["msg_bytes"]
    # bounded: one full step of ONE pipeline per timed step (pipelines are independent and
    # identical; the value scales by the pipeline count, as the GPU arm's does)
    t_one = oracle_step(pp, M, nb)
    steps, warm = args.steps, args.warmup
    if (steps + warm) * t_one > 240:           # keep the whole run within a few minutes
        steps, warm = max(1, int(200 / t_one)), 0
    for _ in range(warm):
        oracle_step(pp, M, nb)
    t = sum(oracle_step(pp, M, nb) for _ in range(steps))
    value = tokens * steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config_dict(wl, world),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                             "sample": f"{steps} full {wl['name']} oracle steps (one pipeline "
                                       f"each, x{wl['pipelines']} pipelines), single process",
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if steps != args.steps:
        line["steps_timed"] = steps
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
class Ctx:
    """Process-level state of the GPU arm."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        import paper_2602_18007_b200 as ppc
        self.torch, self.dist, self.ppc = torch, dist, ppc
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.distributed = self.world > 1
        if self.distributed:
            # one GPU per rank; with fewer GPUs than ranks (a rehearsal of the 8-GPU path on a
            # 4-GPU box) ranks share GPUs round-robin — the numbers are then not a bench line
            self.shared_gpus = self.world > torch.cuda.device_count()
            torch.cuda.set_device(self.local % torch.cuda.device_count())
            dist.init_process_group("gloo")
        else:
            self.shared_gpus = False
            torch.cuda.set_device(0)
        self.dev = torch.cuda.current_device()

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.distributed:
            self.dist.barrier()

    def max_over_ranks(self, v):
        if not self.distributed:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, v):
        if not self.distributed:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64)
        self.dist.all_reduce(t)
        return float(t.item())

    def all_true(self, b):
        return self.sum_over_ranks(0.0 if b else 1.0) == 0.0


class Pipeline:
    """This process's stages of one workload: comms, device buffers X / G / Y / DX, streams,
    step args, optional CUDA graph."""

    def __init__(self, ctx, wl, local_direct=True):
        torch, ppc = ctx.torch, ctx.ppc
        self.ctx, self.wl = ctx, wl
        os.environ["PPC_LOCAL_DIRECT"] = "1" if local_direct else "0"
        S, nb, M = wl["pp"], wl["msg_bytes"], wl["M"]
        engine = {"sm": ppc.ENGINE_SM, "ce": ppc.ENGINE_CE, "pull": ppc.ENGINE_PULL}[wl["engine"]]
        cfg = ppc.make_config(tp=wl["tp"], pp=S, dp=wl["dp"], max_msg_bytes=nb,
                              ring_slots=wl["slots"], channels=wl["channels"],
                              chunk_bytes=wl["chunk"], engine=engine,
                              cta_per_channel=wl["cta"], trace=3)
        if ctx.distributed:
            self.comms = [ppc.connect_distributed(cfg, ctx.rank, ctx.world, ctx.dev,
                                                  with_nccl=wl["tp"] > 1)]
            self.stages = [self.comms[0].group(ppc.GROUP_PP)[0].index(ctx.rank)]
        else:
            self.comms = ppc.virtual_stages(cfg, ctx.dev)
            self.stages = list(range(S))
        dev = ctx.dev
        bufs = lambda: [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(M)]
        self.X = {s: bufs() for s in self.stages if s == 0}
        self.G = {s: bufs() for s in self.stages if s == S - 1}
        self.Y = {s: bufs() for s in self.stages if s == S - 1}
        self.DX = {s: bufs() for s in self.stages if s == 0}
        for s in self.stages:
            for m in range(M):
                if s in self.X:
                    ppc.fill_payload(self.X[s][m], nb, 42, 0, 0xFF, 0, m)
                if s in self.G:
                    ppc.fill_payload(self.G[s][m], nb, 42, 0, 0xFF, 1, m)
        torch.cuda.synchronize()           # inputs (legacy stream) before the stage streams
        self.args = [ppc.StepArgs(M, nb, nb, x=self.X.get(s), g=self.G.get(s),
                                  y=self.Y.get(s), dx=self.DX.get(s)) for s in self.stages]
        self.streams = [torch.cuda.Stream() for _ in self.stages]
        if ctx.distributed and wl["zc"]:
            ppc.register_tensors(self.comms[0], [t for s in self.stages
                                                 for t in self.X.get(s, []) + self.G.get(s, [])])
        self.graph = None
        self.step(eager=True)              # allocates the step buffers
        ctx.barrier()
        if wl["graph"]:
            self.graph = ppc.StepGraph(self.comms, self.args, self.streams)

    def step(self, args=None, eager=False):
        ppc = self.ctx.ppc
        if self.graph is not None and args is None and not eager:
            self.graph.launch()
            return
        a = args or self.args
        if self.ctx.distributed:
            ppc.step_1f1b(self.comms[0], a[0], self.streams[0])
        else:
            ppc.step_1f1b_local(self.comms, a, self.streams)

    def timed(self, steps, instrumented=False):
        """K steps between barriers + synchronize; CUDA events on the launch streams (the
        graph replays on streams[0]); max over ranks.  Returns ms for the K steps."""
        torch, ctx = self.ctx.torch, self.ctx
        for c in self.comms:
            c.set_trace(2 if instrumented else 0)
            c.kernel_times(0), c.kernel_times(1)
        sts = self.streams[:1] if (self.graph is not None and not instrumented) else self.streams
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in sts]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in sts]
        ctx.barrier()
        for e, st in zip(ev0, sts):
            e.record(st)
        for _ in range(steps):
            self.step(eager=instrumented)
        for e, st in zip(ev1, sts):
            e.record(st)
        ctx.barrier()
        return ctx.max_over_ranks(max(a.elapsed_time(b) for a, b in zip(ev0, ev1)))

    def outputs_ok(self):
        """Device-side check of every micro-batch after the timed steps: identity stages, so
        the last stage must hold X_m and stage 0 G_m (compared with the pipeline's own
        inputs on the ranks that have them; otherwise with a fresh SplitMix fill)."""
        torch, ppc = self.ctx.torch, self.ctx.ppc
        ok = True
        nb = self.wl["msg_bytes"]
        ref = torch.empty(nb, dtype=torch.uint8, device=self.ctx.dev)
        for s in self.stages:
            for m in range(self.wl["M"]):
                if s in self.Y:
                    ppc.fill_payload(ref, nb, 42, 0, 0xFF, 0, m)
                    ok &= bool(torch.equal(self.Y[s][m], ref))
                if s in self.DX:
                    ppc.fill_payload(ref, nb, 42, 0, 0xFF, 1, m)
                    ok &= bool(torch.equal(self.DX[s][m], ref))
        return self.ctx.all_true(ok)

    def close(self):
        ctx = self.ctx
        ctx.barrier()
        if self.graph is not None:
            self.graph.destroy()
        for c in self.comms:
            c.disconnect()
        if ctx.distributed:
            ctx.dist.barrier()
        for c in self.comms:
            c.destroy()
        os.environ.pop("PPC_LOCAL_DIRECT", None)


def measure(ctx, wl, steps, warmup, local_direct=True):
    """Steady-state K-step timing of one workload; returns the summary and the pipeline."""
    p = Pipeline(ctx, wl, local_direct)
    for _ in range(warmup):
        p.step()
    ctx.barrier()
    ms = p.timed(steps)
    tokens = wl["pipelines"] * wl["M"] * wl["seq"] * steps
    return p, {"value": tokens / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms / steps}


def kernel_roofline(ctx, p, wl, steps, ms_step):
    """Roofline of the dominant kernel (the one that moves the bytes):
      N = 1 direct: copy_kernel, 2B of HBM per launch (read + write);
      N = 1 ring:   push_ws_kernel (slot write) + recv_kernel (copy-out): 2B each;
      N >= 2 zero-copy: recv_kernel (NVLink pull), B per launch;
      N >= 2 ring:  push_ws_kernel (NVLink stores), B per launch.
    achieved = algorithmic bytes per launch / the launch's duration, measured in an
    instrumented eager pass of the same K steps with CUDA events on the launch streams."""
    ppc = ctx.ppc
    nb = wl["msg_bytes"]
    peaks = measured_peaks()
    n_rec0 = [len(c.trace()) for c in p.comms]
    ms_instr = p.timed(steps, instrumented=True)
    send_ms = [t for c in p.comms for t in c.kernel_times(0)]
    recv_ms = [t for c in p.comms for t in c.kernel_times(1)]
    recs = [r for c, n0 in zip(p.comms, n_rec0) for r in c.trace()[n0:] if r["kind"] == 1]
    for c in p.comms:
        c.set_trace(0)
    if not ctx.distributed:
        alg, peak, bound = 2 * nb, peaks.get("hbm_gbs", 6550.0), "hbm"
        peak_src = ("MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)" if "hbm_gbs" in peaks
                    else "fallback 6.55 TB/s")
    else:
        alg, peak, bound = nb, NVLINK_GBPS, "nvlink"
        peak_src = "NVLink 5 nominal 900 GB/s per direction per GPU"
    dom = recv_ms if (ctx.distributed and wl["zc"]) else send_ms
    if not dom:
        return None
    per_launch = ctx.max_over_ranks(statistics.mean(dom))
    roof = {"bound": bound, "peak": peak, "unit": "GB/s", "peak_source": peak_src,
            "alg_bytes_per_launch": alg, "launches_timed": len(dom),
            "event_launch_us": per_launch * 1e3,
            "event_achieved": alg / (per_launch * 1e-3) / 1e9,
            "instrumented_ms_per_step": ms_instr / steps}
    # the same bytes over the headline (un-instrumented) step: every dominant launch of the
    # step, both directions and all of this process's stages, back to back in the step time
    per_step = alg * len(dom) / steps
    roof["step_aggregate"] = {"bytes_per_step": per_step,
                              "achieved": per_step / (ms_step * 1e-3) / 1e9,
                              "frac": per_step / (ms_step * 1e-3) / 1e9 / peak}
    if ctx.distributed and wl["zc"] and recs:
        ph = ctx.max_over_ranks(statistics.mean((r["t_end_ns"] - r["t_start_ns"]) * 1e-3
                                                for r in recs))
        roof["pull_data_phase"] = {"avg_us": ph, "achieved": nb / (ph * 1e-6) / 1e9,
                                   "frac": nb / (ph * 1e-6) / 1e9 / peak, "records": len(recs),
                                   "timing": "%globaltimer in recv_kernel: publication seen -> "
                                             "last CTA done (excludes the wait for the peer)"}
    return roof


def serialized_copy(ctx, wl, steps):
    """N = 1 direct mode with every hand-off copy on ONE transfer queue (PPC_LOCAL_QUEUE=1),
    so copy_kernel launches never overlap: per-launch CUDA events then time the kernel alone
    (the duration ncu's serialised launch list shows).  Returns (us per launch, launches)."""
    os.environ["PPC_LOCAL_QUEUE"] = "1"
    try:
        p = Pipeline(ctx, {**wl, "graph": False})
        p.step()
        p.timed(steps, instrumented=True)
        ms = [t for c in p.comms for t in c.kernel_times(0)]
        p.close()
    finally:
        os.environ.pop("PPC_LOCAL_QUEUE", None)
    return (statistics.median(ms) * 1e3 if ms else None), len(ms)


def e2e_leg(ctx, p, wl, steps):
    """The same step through the C-ABI with pinned HOST X / G in and HOST Y / DX out: the
    host<->device copies run inside the timed region (libppc's staging streams)."""
    torch, ppc = ctx.torch, ctx.ppc
    nb, M = wl["msg_bytes"], wl["M"]
    hb = lambda: [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(M)]
    hX = {s: hb() for s in p.X}
    hG = {s: hb() for s in p.G}
    hY = {s: hb() for s in p.Y}
    hDX = {s: hb() for s in p.DX}
    for s in hX:
        for m in range(M):
            hX[s][m].copy_(p.X[s][m].cpu())
    for s in hG:
        for m in range(M):
            hG[s][m].copy_(p.G[s][m].cpu())
    args = [ppc.StepArgs(M, nb, nb, x=hX.get(s), g=hG.get(s), y=hY.get(s), dx=hDX.get(s))
            for s in p.stages]
    K2 = max(3, min(steps, 10))
    p.step(args)
    ctx.barrier()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in p.stages]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in p.stages]
    for e, st in zip(e0, p.streams):
        e.record(st)
    for _ in range(K2):
        p.step(args)
    for e, st in zip(e1, p.streams):
        e.record(st)
    ctx.barrier()
    ms = ctx.max_over_ranks(max(a.elapsed_time(b) for a, b in zip(e0, e1)))
    h2d = int(ctx.sum_over_ranks((len(hX) + len(hG)) * M * nb))
    d2h = int(ctx.sum_over_ranks((len(hY) + len(hDX)) * M * nb))
    ok = True                       # identity stages: Y_m = X_m, DX_m = G_m, every m
    ref = torch.empty(nb, dtype=torch.uint8, device=ctx.dev)
    for outs, d in ((hY, 0), (hDX, 1)):
        for s in outs:
            for m in range(M):
                ppc.fill_payload(ref, nb, 42, 0, 0xFF, d, m)
                ok &= bool(torch.equal(outs[s][m].to(ctx.dev), ref))
    hin = [b for d in (hX, hG) for bufs in d.values() for b in bufs]
    hout = [b for d in (hY, hDX) for bufs in d.values() for b in bufs]
    roof = host_link_bound(ctx, hin, hout, nb, ms / K2)
    return {"value": wl["pipelines"] * M * wl["seq"] * K2 / (ms * 1e-3), "unit": "tokens/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms / K2,
            "steps": K2, "outputs_checked": ctx.all_true(ok),
            "roofline": roof or pcie_roofline(ctx.world, h2d / ctx.world, d2h / ctx.world, ms / K2)}


def host_link_bound(ctx, hin, hout, nb, ms_step, reps=3):
    """The e2e step's host-link bound measured in the same run on the same pinned buffers:
    every rank copies its step's inputs host->device and its outputs device->host at once
    (two streams, nothing else), all ranks together; best of `reps`, max over ranks."""
    torch = ctx.torch
    try:
        ddst = torch.empty(nb, dtype=torch.uint8, device=ctx.dev)
        dsrc = torch.zeros(nb, dtype=torch.uint8, device=ctx.dev)
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            ctx.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            sa.wait_event(e0)
            sb.wait_event(e0)
            with torch.cuda.stream(sa):
                for h in hin:
                    ddst.copy_(h, non_blocking=True)
            with torch.cuda.stream(sb):
                for h in hout:
                    h.copy_(dsrc, non_blocking=True)
            ea.record(sa)
            eb.record(sb)
            torch.cuda.synchronize()
            t = max(e0.elapsed_time(ea), e0.elapsed_time(eb))
            best = t if best is None else min(best, t)
        ms = ctx.max_over_ranks(best)
        return {"bound": "pcie+host", "bound_ms_per_step": ms, "frac": ms / ms_step,
                "h2d_gbps_per_gpu": len(hin) * nb / (ms * 1e6),
                "d2h_gbps_per_gpu": len(hout) * nb / (ms * 1e6),
                "source": "measured in this run: the step's H2D and D2H copies alone, both "
                          "directions at once on every rank, best of 3, max over ranks"}
    except Exception:
        return None


def p2p_stream_leg(ctx, n=64 << 20, N=16, reps=5):
    """The metric's first half, "stage-boundary P2P GB/s vs NVLink" (BJ target: >= 80 % of
    900 GB/s for messages >= 64 MB): every pipeline's stage 0 streams N messages of n bytes
    to its stage 1 — zero-copy publications (cfg.zc_async) from a registered buffer, one
    batched receive grid for all N (ppc_pp_recv_batch) — timed on the sender's stream from
    the first publication to ppc_pp_wait_consumed (every byte in the receiver's buffers);
    median of `reps`, max over ranks of the time.  PP = 2 pairs only."""
    torch, ppc = ctx.torch, ctx.ppc
    st, _ = b1_pair(ctx.rank, ctx.world)
    cfg = ppc.make_config(pp=2, dp=ctx.world // 2, max_msg_bytes=n, chunk_bytes=256 << 10,
                          zc_async=1)
    comm = ppc.connect_distributed(cfg, ctx.rank, ctx.world, ctx.dev, with_nccl=False)
    src = torch.empty(n, dtype=torch.uint8, device=ctx.dev)
    ppc.fill_payload(src, n, 42, 0, 0, 0, 0)
    torch.cuda.synchronize()
    ppc.register_tensors(comm, [src] if st == 0 else [])
    dsts = [torch.empty(n, dtype=torch.uint8, device=ctx.dev) for _ in range(N)] if st == 1 else []
    s = torch.cuda.Stream()
    times, mb = [], 0
    for rep in range(reps + 1):
        ctx.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if st == 0:
            for i in range(N):
                comm.send(ppc.FWD, src, n, mb=mb + i, stream=s)
            comm.wait_consumed(ppc.FWD, s)
        else:
            comm.recv_batch(ppc.FWD, dsts, n, mb0=mb, stream=s)
        e1.record(s)
        mb += N
        ctx.barrier()
        t = ctx.max_over_ranks(e0.elapsed_time(e1) if st == 0 else 0.0)
        if rep:
            times.append(t)
    # every rank filled `src` with the same payload: each received buffer must equal it
    ok = all(bool(torch.equal(d, src)) for d in dsts)
    ok = ctx.all_true(ok and comm.poll() == 0)
    ctx.barrier()
    comm.disconnect()
    ctx.dist.barrier()
    comm.destroy()
    t = statistics.median(times) * 1e-3
    gbps = N * n / t / 1e9
    return {"bytes": n, "messages": N, "gbps_per_direction": gbps, "frac_of_900": gbps / NVLINK_GBPS,
            "target": ">= 0.80 of 900 GB/s for >= 64 MB (BASELINE.json)", "outputs_checked": ok,
            "how": "zero-copy publications (zc_async) + one batched receive grid per N messages, "
                   "sender-stream CUDA events to ppc_pp_wait_consumed, median of "
                   f"{reps}, max over ranks"}


def b1_pair(rank, world):
    """(stage, rank of the pipeline's stage-0 rank) of `rank` in a PP = 2, TP = 1 grid of
    `world` ranks: rank = pp_i * dp + dp_i, so stage = rank // dp, pipeline = dp_i."""
    dp = world // 2
    return rank // dp, rank % dp


def b1_arm(ctx, wl, steps=3, channels=4, chunk=4 << 20):
    """CPU-Forwarding baseline B1 (libppcb, P:L37/P:L47/P:L163): D2H into a pinned /dev/shm
    ring, per-chunk host flags, H2D at the receiver, `channels` host threads — the same
    1F1B step (identity stages, the headline's buffers) between the two stages of every
    PP = 2 pipeline; N = 1: both virtual stages in this process, one host thread stepping
    them in dependency order.  Host wall clock (the calls block), max over ranks."""
    torch, ppc = ctx.torch, ctx.ppc
    from paper_2602_18007_b200.cpufwd import CpuFwdLink
    if wl["pp"] != 2:
        return None
    nb, M = wl["msg_bytes"], wl["M"]
    dev = ctx.dev
    s = torch.cuda.current_stream()
    X = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(M)]
    G = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(M)]
    OUT = {0: [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(M)],
           1: [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(M)]}
    for m in range(M):
        ppc.fill_payload(X[m], nb, 42, 0, 0xFF, 0, m)
        ppc.fill_payload(G[m], nb, 42, 0, 0xFF, 1, m)
    K = 2
    if ctx.distributed:
        pids = [None] * ctx.world
        ctx.dist.all_gather_object(pids, os.getpid())
        st, lead_rank = b1_pair(ctx.rank, ctx.world)
        lead = pids[lead_rank]
        fwd = CpuFwdLink(f"b1f_{lead}", st == 0, nb, chunk, K, channels, dev)
        bwd = CpuFwdLink(f"b1b_{lead}", st == 1, nb, chunk, K, channels, dev)
        ctx.dist.barrier()
        fwd.connect()
        bwd.connect()
        ctx.dist.barrier()
        ops = ppc.schedule_1f1b(2, st, M)

        def step():
            for kind, m in ops:
                if st == 0:
                    (fwd.send(X[m], nb, m, s) if kind == "F" else bwd.recv(OUT[0][m], nb, m, s))
                else:
                    (fwd.recv(OUT[1][m], nb, m, s) if kind == "F" else bwd.send(G[m], nb, m, s))
        links = [fwd, bwd]
    else:
        tag = os.getpid()
        fs = CpuFwdLink(f"b1f_{tag}", True, nb, chunk, K, channels, dev)
        fr = CpuFwdLink(f"b1f_{tag}", False, nb, chunk, K, channels, dev)
        bs = CpuFwdLink(f"b1b_{tag}", True, nb, chunk, K, channels, dev)
        br = CpuFwdLink(f"b1b_{tag}", False, nb, chunk, K, channels, dev)
        for ln in (fs, fr, bs, br):
            ln.connect()
        links = [fs, fr, bs, br]
        ops = [ppc.schedule_1f1b(2, st, M) for st in (0, 1)]

        def step():
            # one host thread, both stages: run each stage's next op when its input message
            # exists and a send has a free slot (blocking calls never wait on the other stage)
            i = [0, 0]
            sent = {0: 0, 1: 0}                 # per direction
            recvd = {0: 0, 1: 0}
            while i[0] < len(ops[0]) or i[1] < len(ops[1]):
                prog = False
                for stg in (0, 1):
                    if i[stg] >= len(ops[stg]):
                        continue
                    kind, m = ops[stg][i[stg]]
                    d = 0 if kind == "F" else 1
                    is_send = (stg == 0 and d == 0) or (stg == 1 and d == 1)
                    if is_send:
                        if sent[d] - recvd[d] >= K:
                            continue
                        (fs.send(X[m], nb, m, s) if d == 0 else bs.send(G[m], nb, m, s))
                        sent[d] += 1
                    else:
                        if recvd[d] >= sent[d]:
                            continue
                        (fr.recv(OUT[1][m], nb, m, s) if d == 0 else br.recv(OUT[0][m], nb, m, s))
                        recvd[d] += 1
                    i[stg] += 1
                    prog = True
                if not prog:
                    raise RuntimeError("B1 step made no progress")
    step()
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    dt = ctx.max_over_ranks(time.perf_counter() - t0)
    ok = True
    st_here = [0, 1] if not ctx.distributed else [b1_pair(ctx.rank, ctx.world)[0]]
    for m in range(M):
        if 1 in st_here:
            ok &= bool(torch.equal(OUT[1][m], X[m]))
        if 0 in st_here:
            ok &= bool(torch.equal(OUT[0][m], G[m]))
    ctx.barrier()
    for ln in links:
        ln.destroy()
    tokens = wl["pipelines"] * M * wl["seq"] * steps
    return {"impl": f"B1 CPU-Forwarding (libppcb): D2H -> pinned /dev/shm ring -> H2D, "
                    f"{channels} channel threads, {chunk >> 20} MiB chunks, K={K}",
            "value": tokens / dt, "unit": "tokens/s", "ms_per_step": 1e3 * dt / steps,
            "steps": steps, "outputs_checked": ctx.all_true(ok),
            "timing": "host wall clock (blocking calls), max over ranks"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ctx = Ctx()
    torch, ppc = ctx.torch, ctx.ppc
    wl = resolve(args, ctx.world)
    launches0 = ppc.launch_count()

    # ---- headline: K steps, un-instrumented, clocks sampled during the timed region
    p = Pipeline(ctx, wl)
    for _ in range(args.warmup):
        p.step()
    ctx.barrier()
    sampler = ClockSampler(ctx.dev)
    sampler.start()
    l0 = ppc.launch_count()
    ms_total = p.timed(args.steps)
    launches = int(ctx.sum_over_ranks(ppc.launch_count() - l0))
    clocks = sampler.stop()
    ms_step = ms_total / args.steps
    tokens = wl["pipelines"] * wl["M"] * wl["seq"] * args.steps
    value = tokens / (ms_total * 1e-3)
    outputs_ok = p.outputs_ok()
    roof = kernel_roofline(ctx, p, wl, args.steps, ms_step)
    if roof is not None and not ctx.distributed:
        # the copy launches of a step run two at a time (F and B hand-offs overlap) and tile
        # the whole step: their algorithmic bytes over the headline step time is what the
        # kernel class achieves; a launch timed alone is reported beside it
        us, n = serialized_copy(ctx, wl, args.steps)
        agg = roof["step_aggregate"]
        launches_per_step = roof["launches_timed"] / args.steps
        roof.update({"kernel": "ppc::copy_kernel (virtual-stage SIMT hand-off)",
                     "achieved": agg["achieved"],
                     "avg_launch_us": ms_step * 1e3 / launches_per_step,
                     "timed_region": "headline K steps (CUDA graph, CUDA events on the launch "
                                     "stream): every copy_kernel launch of the step, 2B of HBM "
                                     "each, over the step time (launches overlap in pairs)",
                     "serialized": {"launch_us_median": us, "launches": n,
                                    "achieved": roof["alg_bytes_per_launch"] / (us * 1e-6) / 1e9,
                                    "how": "eager steps with every copy on one transfer queue "
                                           "(PPC_LOCAL_QUEUE=1), CUDA events around each launch "
                                           "(they add the event and launch overhead to each "
                                           "launch; ncu_serialized is the kernel alone)"},
                     "traffic": ncu_traffic("copy_n1")})
        ns = ncu_traffic("copy_n1_launch_ns")
        if ns:
            a = roof["alg_bytes_per_launch"] / (ns * 1e-9) / 1e9
            roof["ncu_serialized"] = {"launch_us": ns * 1e-3, "achieved": a, "frac": a / roof["peak"],
                                      "source": "committed ncu launch list of this bench "
                                                "(profiles/ncu_traffic.json copy_n1_launch_ns)"}
    elif roof is not None and wl["zc"]:
        ph = roof.get("pull_data_phase", {})
        roof.update({"kernel": "ppc::recv_kernel (zero-copy NVLink pull into the user buffer)",
                     "achieved": ph.get("achieved", roof["event_achieved"]),
                     "avg_launch_us": ph.get("avg_us", roof["event_launch_us"]),
                     "timed_region": "per-launch data phase (%globaltimer, publication seen -> "
                                     "last CTA); event_* = CUDA events around the launch, "
                                     "which include the wait for the peer's publication",
                     "traffic": ncu_traffic("recv_n2"),
                     "traffic_counters": "ncu nvlrx__bytes_data_user.sum + nvltx__bytes_data_user"
                                         ".sum per launch (profiles/ncu_traffic.json)"})
        nvl = ncu_traffic("recv_n2_nvl_totals")
        if nvl:
            # what an SM pull can reach on these links: every 128-B read costs 16 B of response
            # header (rx) and a 24-B request travelling the other way (tx), so with both
            # directions pulling each link direction carries rx + the reverse pull's tx
            bi = roof["peak"] * nvl["user_bytes"] / (nvl["nvlrx_bytes"] + nvl["nvltx_bytes"])
            uni = roof["peak"] * nvl["user_bytes"] / nvl["nvlrx_bytes"]
            roof["protocol_bound"] = {
                "bidir_gbps": bi, "uni_gbps": uni, "frac_bidir": roof["achieved"] / bi,
                "how": "900 GB/s x user / NVLink bytes (incl. protocol) of one pull, from the "
                       "committed ncu NVLink counters (profiles/ncu_traffic.json)"}
    elif roof is not None:
        roof.update({"kernel": "ppc::push_ws_kernel (SM push over NVLink)",
                     "achieved": roof["event_achieved"], "avg_launch_us": roof["event_launch_us"],
                     "timed_region": "CUDA events around every push launch (instrumented pass)",
                     "traffic": ncu_traffic("push_n2"),
                     "traffic_counters": "ncu nvltx__bytes_data_user.sum + nvlrx__bytes_data_user"
                                         ".sum per launch (profiles/ncu_traffic.json)"})
    if roof is not None:
        roof["frac"] = roof["achieved"] / roof["peak"]

    e2e = None if args.no_e2e else e2e_leg(ctx, p, wl, args.steps)
    p.close()

    # ---- N = 1: the intra-device ring (push into the slot + chunk flags + copy-out)
    ring = None
    if not ctx.distributed and not args.no_ring:
        pr, ring = measure(ctx, wl, args.steps, args.warmup, local_direct=False)
        ring["outputs_checked"] = pr.outputs_ok()
        rr = kernel_roofline(ctx, pr, wl, args.steps, ring["ms_per_step"])
        pr.close()
        ring["config"] = "PPC_LOCAL_DIRECT=0: push_ws_kernel writes the ring slot (chunk flags), " \
                         "recv_kernel copies it out; CUDA graph"
        if rr:
            ring["roofline"] = {k: rr[k] for k in ("bound", "peak", "unit", "step_aggregate",
                                                   "event_launch_us", "event_achieved")}
            # every message moves 4B of HBM on the ring (slot write + copy-out)
            msgs = 2 * wl["M"]
            ring["hbm_gbps_step"] = 4 * wl["msg_bytes"] * msgs / (ring["ms_per_step"] * 1e-3) / 1e9
            ring["hbm_frac_step"] = ring["hbm_gbps_step"] / rr["peak"]

    # ---- north-star configurations beside the headline (as many as the GPUs allow)
    extra = {}
    if not args.no_extra:
        for name in EXTRA.get(ctx.world, []):
            wx = resolve(args, ctx.world, name)
            try:                        # a side measurement must not sink the headline line
                px, r = measure(ctx, wx, max(3, args.steps // 2), max(3, args.warmup))
                r["outputs_checked"] = px.outputs_ok()
                px.close()
            except Exception as e:
                r = {"error": repr(e)[:300]}
            r["config"] = config_dict(wx, ctx.world)
            extra[name] = r

    # ---- stage-boundary P2P GB/s (the metric's first half), N >= 2
    p2p = None
    if ctx.distributed and not ctx.shared_gpus and ctx.world % 2 == 0:
        try:
            p2p = p2p_stream_leg(ctx)
        except Exception as e:
            p2p = {"error": repr(e)[:200]}

    # ---- CPU-Forwarding B1 on the headline workload
    b1 = None
    if not args.no_b1:
        try:
            b1 = b1_arm(ctx, wl)
        except Exception as e:          # the baseline must not sink the line
            b1 = {"error": repr(e)[:200]}

    cpu = None
    if ctx.rank == 0 and not ctx.distributed and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": config_dict(wl, ctx.world), "outputs_checked": outputs_ok,
            "boundary_gbps": 2 * wl["M"] * wl["msg_bytes"] * wl["pipelines"] * (wl["pp"] - 1)
                             / (ms_step * 1e-3) / 1e9,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches, "cpu_forwarding": b1,
        }
        if b1 and "value" in b1:
            line["device_direct_vs_cpu_forwarding"] = value / b1["value"]
        if ring:
            line["intra_device_ring"] = ring
        if p2p:
            line["p2p_stream_64MiB"] = p2p
        if extra:
            line["north_star_configs"] = extra
        if ctx.shared_gpus:
            line["shared_gpus"] = ("REHEARSAL: more ranks than GPUs, ranks share GPUs "
                                   "(time-sliced); not a bench line")
        if ctx.distributed and wl["pp"] == 2:
            t_msg = wl["msg_bytes"] / (NVLINK_GBPS * 1e3)
            line["step_roofline"] = {"us": (wl["M"] + 1) * t_msg,
                                     "frac": (wl["M"] + 1) * t_msg / (ms_step * 1e3),
                                     "model": "PP2 comm-only critical path (M+1) x t_msg at "
                                              "900 GB/s (DESIGN.md R5; oracle O2)"}
        print(json.dumps(line), flush=True)
    ctx.barrier()
    if ctx.distributed:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()

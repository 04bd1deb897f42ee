#!/usr/bin/env python
"""Benchmark of the KAN-layer forward hot path (BASELINE.json metric:
"KAN samples/sec (int8-LUT path) and % of roofline at 1/2/4/8 B200").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A step = one forward pass of the workload over its GLOBAL batch.  Default
workload = BASELINE.json configs[4] (C5), the config the metric is quoted on
at 1/2/4/8 GPUs: ResKAN18 on 3x32x32, G=5, P=3, 3-bit table (k=8, h=3),
8-bit weights in the reference's own per-tensor asymmetric scheme, no SiLU
term, fp32 logits, global batch 8192 -- the arithmetic the reference's CPU
path (`--impl reference`) computes, so both arms print the same `config`.
`--config c5pc` is the same network with per-channel int8 W + SiLU; c1..c4,
c3bf16 and the spline-table variants select the other BASELINE configs.

Multi-GPU: one process per GPU (torchrun; `--gpus N` without
torchrun re-launches itself under torch.distributed.run).  The global batch is
split into contiguous shards (strong scaling: 8192/N rows per GPU); each rank
forwards its shard with no collective, and the logits are gathered to rank 0
over NCCL inside the timed region, every step.

Timing: W untimed warm-up steps, then exactly K steps bracketed by a barrier
and cudaDeviceSynchronize on both sides, device-timed with CUDA events on the
launching stream, max over ranks.  Inputs rotate over resident batches whose
total exceeds the 126 MB L2 (C5 also writes >2 GB of intermediates per step).
Small-batch configs (C1/C2) keep several batches in flight on separate
streams: the timed region replays CUDA graphs holding exactly K forwards.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
# independent batches in flight per GPU for the latency-bound small configs
# (one engine + CUDA stream each; bench.py --streams overrides)
STREAMS_DEFAULT = {"c1": 20, "c2": 12, "c1st": 4, "c2st": 4, "c2st4": 4}
# K splits per launch (0 = the engine's choice)
SPLIT_DEFAULT = {"c1": 1, "c2": 1}
PAPER_SAMPLES_PER_S = {  # PAPER.md:603, KANMLP2 G=5 8-bit LUT on RTX 3090
    "c1": 10000 / 5.9e-3, "c2": 10000 / 5.9e-3,
}
GRAPH_CHUNK = 1000  # forwards per captured graph (small configs)


def per_config(table, key, default):
    """A per-config default; sweep variants (c2k4, c1fp32, ...) inherit their base config's."""
    return table.get(key, table.get(key[:2], default))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="wall time of the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--streams", type=int, default=0,
                    help="batches in flight (one engine + stream each); 0 = per-config default")
    ap.add_argument("--split-k", type=int, default=0, help="force the K splits of split-K launches")
    ap.add_argument("--opt", action="append", default=[],
                    help="engine tuning option name=value (kan_engine_set_option; experiments only)")
    return ap.parse_args()


def relaunch_under_torchrun(args):
    """--gpus N > 1 outside torchrun: re-run this command as N ranks (one per GPU)."""
    port = 29500 + (os.getpid() % 1000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def world_info(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    return world, rank, local


def shard(batch, rank, world):
    per = (batch + world - 1) // world
    s = min(batch, rank * per)
    return s, min(batch, s + per)


def line_config(wl, world):
    """The `config` object both arms print (identical on the same workload)."""
    return {"workload": wl.key + ": " + wl.title, "scheme": wl.scheme(), "global_batch": wl.batch,
            "batch_per_gpu": (wl.batch + world - 1) // world, "parallelism": f"dp{world}",
            "l2": "inputs rotate over resident batches larger than the 126 MB L2"}


def metric_name(wl):
    if wl.mode == "bspline-lut":
        return "KAN samples/sec (int8-LUT path)"
    return f"KAN samples/sec ({wl.mode} path)"


# ---------------------------------------------------------------------------------
class ClockSampler:
    """NVML sampling of SM clocks and clock-event reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.ok = False
        self.samples = []
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self._phys(device))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    @staticmethod
    def _phys(device):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[device])
            except (ValueError, IndexError):
                return device
        return device

    def _read(self):
        nv = self.nv
        mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        return (time.perf_counter(), mhz, rs)

    def start(self):
        if not self.ok:
            return
        self._stop = False
        self.samples.append(self._read())

        def loop():
            while not self._stop:
                try:
                    self.samples.append(self._read())
                except Exception:
                    pass
                time.sleep(0.002)
        self.th = threading.Thread(target=loop, daemon=True)
        self.th.start()

    def stop(self):
        if not self.ok:
            return
        self._stop = True
        self.th.join()
        self.samples.append(self._read())

    def summary(self, t0, t1):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        inside = [s for s in self.samples if t0 <= s[0] <= t1] or self.samples
        mhz = sorted(s[1] for s in inside)
        mask = 0
        for s in inside:
            mask |= s[2]
        reasons = [n for b, n in self.REASONS.items() if mask & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(mhz)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(inside)}


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"), "/root/repo/MEASURED_PEAKS.json"):
        if os.path.exists(p):
            with open(p) as f:
                return json.load(f), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


def measure_int8_peak(dev):
    """Dense int8 tensor-core peak on this box: cuBLASLt int8 GEMM through
    torch._int_mm, 8192^3, best of 10 (CUDA events).  None if unavailable."""
    import torch
    try:
        n = 8192
        a = torch.randint(-127, 127, (n, n), device=dev, dtype=torch.int8)
        b = torch.randint(-127, 127, (n, n), device=dev, dtype=torch.int8).t().contiguous().t()
        for _ in range(3):
            torch._int_mm(a, b)
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2 * n ** 3 / (best / 1e3) / 1e12
    except Exception:
        return None


def committed_traffic(key: str, kernel, layers):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    captures (profiles/ncu_summary.json): the average over all of the kernel's
    launches of a forward ("<workload>_<kernel>": one ncu pass over every launch),
    or the capture of the single KAN layer ("<workload>_l<layer>"); None without one."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    if kernel is not None and len(layers) > 1:
        return d.get(f"{key}_{kernel}", {}).get("dram_bytes_per_launch")
    return d.get(f"{key}_l{layers[0]}", {}).get("dram_bytes_per_launch")


# ---------------------------------------------------------------------------------
def ref_forward(ref, wl, Ws, x, threads):
    """One call of the reference's CPU path on rows x: model_forward for models
    the reference's descriptor schema expresses (bspline-lut mode, per-tensor u8
    W, eval.hpp:70-76, no SiLU term -- the reference has none); for ResKAN18 the
    harness composition of reference functions (oracle/ref_shim.cpp
    ref_graph_forward: convkan_forward + residual adds + pooling)."""
    text = json.dumps(wl.descriptor())
    if wl.reference_expressible:
        return ref.model_forward(text, Ws, x, wl.out_size, mode=2, k=wl.lut_k, h=wl.lut_h,
                                 bits_w=8, threads=threads, chunk=256)
    return ref.graph_forward(text, Ws, x, wl.out_size, k=wl.lut_k, h=wl.lut_h, bits_w=8,
                             threads=threads)


def cpu_rows(wl, cores):
    """Rows per reference call: 256-row chunks per thread for the MLPs; for the
    conv models (0.6-9 GOP per sample) one sample per thread."""
    return 256 * cores if wl.layers is None else cores


def reference_sample(wl, seconds: float, threads: int):
    """Time the reference's own CPU path (oracle/_ref: the reference headers
    compiled unmodified) on a bounded sample of the workload; returns
    (samples/s, description).  Falls back to the C restatement (1 thread)."""
    from oracle.pyoracle import Oracle, Ref
    Ws, _ = wl.weights()
    rows = cpu_rows(wl, threads)
    x = wl.inputs(rows, seed=99).astype(np.float64)
    if Ref.available and wl.mode == "spline-table":
        ref = Ref()
        text = json.dumps(wl.descriptor())
        n, dt = 0, 0.0
        while dt < seconds:
            _, sec = ref.st_model_forward(text, Ws, x, wl.out_size, wl.lut_k, wl.lut_h,
                                          threads=threads, chunk=256)
            n += rows
            dt += sec
        return n / dt, threads, "reference", (
            f"{n} samples ({rows}-row calls) through the reference model_forward in spline-table mode "
            f"(tables built once, untimed), {threads} threads, {dt:.1f} s")
    if Ref.available:
        ref = Ref()
        n = 0
        t0 = time.perf_counter()
        while True:
            ref_forward(ref, wl, Ws, x, threads)
            n += rows
            if time.perf_counter() - t0 >= seconds:
                break
        dt = time.perf_counter() - t0
        how = ("model_forward" if wl.reference_expressible else
               "convkan_forward/kan_linear_forward composition (ref_graph_forward)")
        return n / dt, threads, "reference", (
            f"{n} samples ({rows}-row calls) through the reference {how}, bspline-lut k{wl.lut_k} "
            f"h{wl.lut_h}, per-tensor u8 W, no SiLU, {threads} threads, {dt:.1f} s")
    if wl.layers is not None:
        raise RuntimeError("oracle/_ref not built: no CPU baseline for conv models")
    o = Oracle()
    g = o.grid(wl.G, wl.P)
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        h = x[:256]
        for w in Ws:
            h = o.lut_forward(g, wl.lut_k, wl.lut_h, 8, h, w)
        n += 256
    dt = time.perf_counter() - t0
    return n / dt, 1, "port", f"{n} samples through the C restatement, 1 thread, {dt:.1f} s"


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path on the
    host cores, on the same workload / metric / config as our arm.  Under
    torchrun only rank 0 runs; the others exit 0 without work.  This arm never
    imports the engine (configs is pure numpy; the package loads libkan_b200.so
    only when an engine name is touched)."""
    world, rank, _ = world_info(args)
    if rank != 0:
        return
    from paper_2603_17230_b200 import configs
    from oracle.pyoracle import Ref
    wl = configs.get(args.config)
    cores = os.cpu_count() or 1
    if not Ref.available:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference headers) not built"}))
        return
    if not wl.reference_scheme and wl.mode != "spline-table":
        note = ("the reference computes per-tensor u8 W without a SiLU term; this workload's scheme "
                "differs, so the reference arm runs the reference scheme on the same shapes")
    else:
        note = "same arithmetic as the GPU arm (the reference's own scheme)"
    rows = cpu_rows(wl, cores)
    x = wl.inputs(rows, seed=7).astype(np.float64)
    Ws, _ = wl.weights()
    ref = Ref()
    st_mode = wl.mode == "spline-table"
    text = json.dumps(wl.descriptor())

    def step():
        if st_mode:
            return ref.st_model_forward(text, Ws, x, wl.out_size, wl.lut_k, wl.lut_h,
                                        threads=cores, chunk=256)[1]
        t = time.perf_counter()
        ref_forward(ref, wl, Ws, x, cores)
        return time.perf_counter() - t
    for _ in range(args.warmup):
        step()
    dt = 0.0
    for _ in range(args.steps):
        dt += step()
    v = rows * args.steps / dt
    print(json.dumps({
        "impl": "reference", "metric": metric_name(wl), "value": v, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": line_config(wl, world),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} steps x {rows} rows (a bounded sample of the global batch), "
                                   f"{cores} threads, after {args.warmup} warm-up steps"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "notes": {"path": ("reference model_forward" if wl.reference_expressible else
                           "reference convkan_forward/kan_linear_forward composition (ref_graph_forward)")
                  + f" from oracle/_ref, {note}"},
    }))


# ---------------------------------------------------------------------------------
def build_engines(wl, dev_index, n, opts, options=()):
    from paper_2603_17230_b200 import Engine
    Ws, Bs = wl.weights()
    out = []
    for _ in range(n):
        e = Engine(wl.descriptor(), dev_index)
        for i, (w, b) in enumerate(zip(Ws, Bs)):
            e.set_coeffs(i, w, b)
        for kv in options:
            k, v = kv.split("=")
            e.set_option(k, int(v))
        e.configure(opts)
        out.append(e)
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2603_17230_b200 import EvalOptions, OUT_I8, configs
    from paper_2603_17230_b200.sharding import LogitGather

    world, rank, local = world_info(args)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    wl = configs.get(args.config)
    r0, r1 = shard(wl.batch, rank, world)
    B = r1 - r0  # this rank's shard (strong scaling)
    per = (wl.batch + world - 1) // world

    n_streams = max(1, args.streams or per_config(STREAMS_DEFAULT, wl.key, 1))
    opts = EvalOptions(**wl.eval_options(), split_k=args.split_k or per_config(SPLIT_DEFAULT, wl.key, 0))
    engines = build_engines(wl, local, n_streams, opts, args.opt)
    eng = engines[0]

    # rotating resident input shards, total > 2x L2
    in_bytes = B * wl.input_size * 4
    R = max(2, min(64, math.ceil(2 * L2_BYTES / max(in_bytes, 1))))
    R = max(R, n_streams)
    xs = [torch.from_numpy(wl.inputs(wl.batch, seed=100 + r)[r0:r1]).to(dev) for r in range(R)]
    if wl.int8_out:  # calibrate the int8 logit scale once (outside the timed region)
        y = eng.model_forward(xs[0]).float()
        opts.out_kind, opts.out_scale = OUT_I8, float(y.abs().max().item()) / 127.0
        for e_ in engines:
            e_.configure(opts)
    out_dtype = torch.int8 if wl.int8_out else torch.float32
    outs = torch.empty((R, B, wl.out_size), device=dev, dtype=out_dtype)
    st = torch.cuda.Stream(dev)
    streams = [st] + [torch.cuda.Stream(dev) for _ in range(n_streams - 1)]
    lg = LogitGather(wl.batch, wl.out_size, out_dtype, dev) if world > 1 else None

    def gather(r):
        """logits of input r to rank 0 over NCCL (padded equal shards)."""
        return lg(outs[r])

    eng.set_option("record_plan", 1)
    with torch.cuda.stream(st):
        for k, e_ in enumerate(engines):
            for r in range(R):
                e_.model_forward(xs[r], out=outs[r], stream=st)
    torch.cuda.synchronize()
    plan = eng.last_plan
    eng.set_option("record_plan", 0)
    launches_per_step = eng.last_launches

    small = n_streams > 1
    graphs = {}

    def graph_of(n_fw, start):
        """CUDA graph of n_fw forwards, forward i on stream i % n_streams (its own
        engine), inputs rotating from `start`; forked from / joined into st."""
        key = (n_fw, start % R)
        if key not in graphs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for s_ in streams[1:]:
                    s_.wait_stream(st)
                for i in range(n_fw):
                    k = i % n_streams
                    r = (start + i) % R
                    engines[k].model_forward(xs[r], out=outs[r], stream=streams[k])
                for s_ in streams[1:]:
                    st.wait_stream(s_)
            graphs[key] = g
        return graphs[key]

    fwd_graphs = {}

    def fwd_graph(r):
        """CUDA graph of one forward of resident input r (big configs: a step
        is one graph replay, so host launch work stays off the device clock)."""
        if r not in fwd_graphs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                engines[0].model_forward(xs[r], out=outs[r], stream=st)
            fwd_graphs[r] = g
        return fwd_graphs[r]

    def run_steps(n, start=0):
        """Exactly n forwards (steps) of this rank's shard, each followed by the
        logit gather to rank 0 (small configs: one gather per replayed graph,
        covering every forward in it)."""
        done = 0
        while done < n:
            if small:
                c = min(GRAPH_CHUNK, n - done)
                graph_of(c, start + done).replay()
                if world > 1:
                    for i in range(c):
                        gather((start + done + i) % R)
                done += c
            else:
                r = (start + done) % R
                fwd_graph(r).replay()
                if world > 1:
                    gather(r)
                done += 1

    with torch.cuda.stream(st):
        run_steps(args.warmup)
        if not small:
            for r in range(R):  # every step's graph exists before the timed region
                fwd_graph(r)
        if small:
            graph_of(min(GRAPH_CHUNK, args.steps), args.warmup)
            if args.steps % GRAPH_CHUNK and args.steps > GRAPH_CHUNK:
                graph_of(args.steps % GRAPH_CHUNK, args.warmup + args.steps - args.steps % GRAPH_CHUNK)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    t_wall0 = time.perf_counter()
    with torch.cuda.stream(st):
        ev0.record(st)
        run_steps(args.steps, args.warmup)
        ev1.record(st)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = wl.batch * args.steps / (ms / 1e3)

    # ---- dominant kernel: per-launch device time with CUDA events (engine profiling:
    # an event pair around each KAN layer's kernel node, replayed from a graph)
    prof_steps = max(2, min(args.steps, 64 if B * wl.input_size < 2 ** 24 else 8))
    eng.set_profiling(True)
    pg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(pg, stream=st):
        for i in range(prof_steps):
            eng.model_forward(xs[i % R], out=outs[i % R], stream=st)
    pg.replay()
    torch.cuda.synchronize()
    layer_ms = []
    for li in range(wl.n_kan):
        tot, cnt = eng.layer_time_ms(li)
        layer_ms.append(tot / max(cnt, 1))
    eng.set_profiling(False)
    # one batch alone, graph-replayed (the latency of a single forward)
    sg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(sg, stream=st):
        eng.model_forward(xs[0], out=outs[0], stream=st)
    sg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(10):
            sg.replay()
        e1.record(st)
    torch.cuda.synchronize()
    single_ms = e0.elapsed_time(e1) / 10
    # the same single batch at the engine's automatic split (small configs: the
    # layer-0 tiles spread over a cluster per tile, the output layer fused into
    # the reduction, one launch): the latency a caller with one batch sees
    single_auto_ms = None
    if n_streams > 1 and opts.split_k != 0:
        o2 = EvalOptions(**{**vars(opts), "split_k": 0})
        ea = build_engines(wl, local, 1, o2, args.opt)[0]
        ea.model_forward(xs[0], out=outs[0], stream=st)
        torch.cuda.synchronize()
        ag = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ag, stream=st):
            ea.model_forward(xs[0], out=outs[0], stream=st)
        ag.replay()
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(10):
                ag.replay()
            e1.record(st)
        torch.cuda.synchronize()
        single_auto_ms = e0.elapsed_time(e1) / 10
        del ea

    lut = wl.mode == "bspline-lut"
    st_mode = wl.mode == "spline-table"
    peaks, peak_src = measured_peaks()
    # per-layer algorithmic bytes.  Residual blocks (the engine's descriptor
    # extension): the launch plan says how a layer's tensors are stored -- a block
    # output kept as fp32 values (epi=0) with its u16 levels sidecar (lv=1), and
    # the fp32 residual it adds (res=2) -- so the algorithmic bytes count them too
    layer_kernel = {}
    layer_bytes = [wl.layer_bytes_per_launch(li, B) for li in range(wl.n_kan)]
    for ln in plan.strip().splitlines():
        f = dict(kv.split("=") for kv in ln.split()[1:])
        li = int(f.get("layer", -1))
        name = ln.split()[0]
        if li < 0 or name in ("im2col_levels", "nchw_to_nhwc", "level_prepass"):
            continue
        layer_kernel[li] = name  # the layer's contraction kernel
        if lut and name in ("convw", "conv3", "gather"):
            kl = wl.kan_layers()[li]
            if li != wl.n_kan - 1:
                out_b = (4 if f["epi"] == "0" else 2) + (2 if f["lv"] == "1" else 0) + (4 if f["res"] == "2" else 0)
                layer_bytes[li] += B * kl["out_elems"] * (out_b - 2)  # layer_bytes_per_launch counted u16 levels out
            elif f["res"] == "2":
                layer_bytes[li] += B * kl["out_elems"] * 4
    # the dominant kernel: the kernel function with the largest share of the step
    # (ResKAN18: kan_convw, 15 launches per forward); its roofline averages over
    # its launches (algorithmic work of all of them / their total duration), and
    # the slowest single launch is reported next to it
    groups = {}
    for li in range(wl.n_kan):
        groups.setdefault(layer_kernel.get(li, "layer"), []).append(li)
    dom_name = max(groups, key=lambda k: sum(layer_ms[li] for li in groups[k]))
    dom_layers = groups[dom_name]
    dom = max(dom_layers, key=lambda li: layer_ms[li])  # its slowest launch
    n_l = len(dom_layers)
    bytes_l = sum(layer_bytes[li] for li in dom_layers) / n_l
    ops_l = sum(wl.layer_ops_per_launch(li, B) for li in dom_layers) / n_l
    t_ms = sum(layer_ms[li] for li in dom_layers) / n_l
    if small:
        # several batches in flight: per-launch event brackets cannot isolate one
        # launch, so the unit is the whole forward over the effective time per batch
        bytes_l = (B * wl.input_size * 4 + B * wl.out_size * (1 if wl.int8_out else 4)
                   + sum(wl.weight_bytes(li) for li in range(wl.n_kan)))
        ops_l = wl.ops_per_sample() * B
        t_ms = ms / args.steps
        layer_ms[dom] = t_ms
    int8_peak, int8_src = None, None
    if lut:
        int8_peak = measure_int8_peak(dev)
        int8_src = "measured in this run: torch._int_mm (cuBLASLt) int8 8192^3, best of 10"
        if int8_peak is None:
            int8_peak, int8_src = 4500.0, "datasheet 4.5 POPS dense int8 (measurement failed)"
    tensor_peak = (int8_peak if lut else peaks.get("bf16_tflops", 1661.3)) * 1e12
    hbm_peak = peaks["hbm_gbs"] * 1e9

    def roof_of(ops, nbytes, t_s):
        if st_mode or ops / nbytes < tensor_peak / hbm_peak:
            r = {"bound": "hbm", "achieved": nbytes / t_s / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
        else:
            r = {"bound": "tensor", "achieved": ops / t_s / 1e12, "peak": tensor_peak / 1e12,
                 "unit": "TOP/s" if lut else "TFLOP/s"}
        r["frac"] = r["achieved"] / r["peak"]
        return r

    def layer_name(li):
        kl = wl.kan_layers()[li]
        return (f"KAN layer {li} ({kl['n_in']}->{kl['n_out']}" + (f", {kl['pix']} px/sample)" if kl["pix"] > 1 else ")"))

    kfn = {"convw": "kan_convw_kernel", "conv3": "kan_conv3_kernel", "gather": "kan_gather_gemm_kernel",
           "gather_bf16": "kan_gather_gemm_kernel (bf16)", "small_layer": "kan_small_layer_kernel"}.get(dom_name, dom_name)
    roof = roof_of(ops_l, bytes_l, t_ms / 1e3)
    roof["traffic"] = committed_traffic(wl.key, dom_name, dom_layers) if not small else None
    if small:
        roof["kernel"] = f"whole forward ({launches_per_step} launch(es) per batch, {n_streams} batches in flight)"
    elif n_l == 1:
        roof["kernel"] = f"{kfn}: " + layer_name(dom)
    else:
        roof["kernel"] = (f"{kfn}: {n_l} launches per forward (KAN layers "
                          + ",".join(str(li) for li in dom_layers) + "), averaged over its launches")
    roof["per_launch"] = {"algorithmic_bytes": bytes_l, "algorithmic_ops": ops_l, "avg_ms": t_ms,
                          "launches_per_forward": 1 if small else n_l,
                          "launches_timed": prof_steps * (1 if small else n_l),
                          "timing": ("timed region / steps (batches in flight)" if small
                                     else "CUDA event pair around each kernel node, graph replay")}
    roof["peak_source"] = (int8_src if lut and roof["bound"] == "tensor" else peak_src)
    roof["layer_avg_ms"] = layer_ms
    # share of the forward, from the same per-launch brackets (their sum runs a few
    # percent above the timed step: bracketed launches do not overlap their tails)
    roof["share_of_step"] = 1.0 if small else t_ms * n_l / max(sum(layer_ms), 1e-12)
    if not small and n_l > 1:
        sl = roof_of(wl.layer_ops_per_launch(dom, B), layer_bytes[dom], layer_ms[dom] / 1e3)
        roof["slowest_launch"] = {"kernel": layer_name(dom), "avg_ms": layer_ms[dom], "frac": sl["frac"],
                                  "achieved": sl["achieved"], "algorithmic_bytes": layer_bytes[dom],
                                  "algorithmic_ops": wl.layer_ops_per_launch(dom, B),
                                  "traffic": committed_traffic(wl.key, None, [dom])}
    # whole-forward tensor roofline (every KAN layer's dense contraction)
    whole = {"ops_per_sample": wl.ops_per_sample(), "achieved": value * wl.ops_per_sample() / 1e12 / world,
             "unit": "TOP/s per GPU" if lut else "TFLOP/s per GPU"}
    whole["frac"] = whole["achieved"] / (tensor_peak / 1e12)

    # ---- e2e through the public API: host buffers, H2D + forward + D2H every step
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(4, min(args.steps, 300 if small else 20))
        hx = [torch.from_numpy(wl.inputs(wl.batch, seed=500 + r)[r0:r1]).pin_memory() for r in range(2)]
        if world == 1:
            # two host threads with their own engine + stream, so one call's H2D
            # overlaps the other's forward (kan_engine_forward_host releases the GIL)
            n_e2e = 2
            e2e_engines = list(engines[:n_e2e])
            if len(e2e_engines) < n_e2e:
                e2e_engines += build_engines(wl, local, n_e2e - len(e2e_engines), opts, args.opt)
            e2e_streams = [torch.cuda.Stream(dev) for _ in range(n_e2e)]
            houts = [torch.empty((B, wl.out_size), dtype=out_dtype).pin_memory() for _ in range(n_e2e)]
            e2e_steps -= e2e_steps % n_e2e

            def e2e_worker(k, n):
                for i in range(n):
                    e2e_engines[k].forward_host_ptr(hx[(i + k) % 2].data_ptr(), B, houts[k].data_ptr(),
                                                    stream=e2e_streams[k])
            for k in range(n_e2e):
                e2e_worker(k, 2)
            t0 = time.perf_counter()
            ths = [threading.Thread(target=e2e_worker, args=(k, e2e_steps // n_e2e)) for k in range(n_e2e)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            e2e_s = time.perf_counter() - t0
            api = "kan_engine_forward_host (pinned host buffers; 2 host threads, one engine + stream each)"
        else:
            # each rank: H2D of its shard, forward, NCCL gather to rank 0, D2H there
            xd = torch.empty_like(xs[0])
            hout = torch.empty((wl.batch, wl.out_size), dtype=out_dtype).pin_memory()

            def e2e_step(i):
                with torch.cuda.stream(st):
                    xd.copy_(hx[i % 2], non_blocking=True)
                    eng.model_forward(xd, out=outs[0], stream=st)
                    full = gather(0)
                    if rank == 0:
                        hout.copy_(full, non_blocking=True)
                st.synchronize()
            for i in range(2):
                e2e_step(i)
            dist.barrier()
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                e2e_step(i)
            e2e_s = time.perf_counter() - t0
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
            api = "Engine.model_forward (kan_engine_forward) + NCCL gather of logits to rank 0, pinned host buffers"
        e2e = {"value": wl.batch * e2e_steps / e2e_s, "unit": "samples/s",
               "h2d_bytes_per_step": wl.batch * wl.input_size * 4,
               "d2h_bytes_per_step": wl.batch * wl.out_size * (1 if wl.int8_out else 4),
               "steps": e2e_steps, "api": api}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, kind, sample = reference_sample(wl, args.cpu_seconds, os.cpu_count() or 1)
            cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": kind, "sample": sample}
        except Exception as ex:  # report, never hide
            cpu = {"value": None, "error": str(ex)}

    if rank == 0:
        paper = PAPER_SAMPLES_PER_S.get(wl.key)
        line = {
            "metric": metric_name(wl),
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": (value / paper) if paper else None,
            "dtype": "u8" if (lut or st_mode) else wl.mode, "data": "synthetic",
            "config": line_config(wl, world),
            "roofline": roof, "whole_forward": whole, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(t_wall0, t_wall1),
            "timing": {"streams": n_streams, "split_k": opts.split_k or "auto", "engine_options": args.opt,
                       "concurrency": (f"{n_streams} batches in flight (one engine + CUDA stream each); "
                                       f"CUDA graphs holding exactly {args.steps} forwards"
                                       if small else "one batch at a time, one CUDA-graph replay per step"),
                       "inputs": f"rotate over {R} resident shards ({R * in_bytes / 2**20:.0f} MiB)",
                       "single_batch_ms": single_ms,
                       "single_batch_auto_split_ms": single_auto_ms,
                       "gather": "NCCL gather of every step's logits to rank 0" if world > 1 else None,
                       "launch_plan": plan.strip().splitlines(),
                       "vs_baseline_ref": ("PAPER.md:603 KANMLP2 G=5 8-bit LUT, RTX 3090, 1.69M samples/s"
                                           if paper else None)},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the KAN-layer forward hot path (BASELINE.json metric:
"KAN samples/sec (int8-LUT path) and % of roofline at 1/2/4/8 B200").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
                  [--streams S] [--split-k K]

A step = one forward pass of the workload over one batch of synthetic input.
Default workload = BASELINE.json configs[1] (C2): KAN MLP [784,64,10], G=5,
P=3, batch 4096 per GPU, 8-bit table (k=8, h=8), int8 per-channel weights,
SiLU base term, hidden outputs requantized to the next layer's lattice, int8
logits.  For N > 1 (torchrun, one process per GPU, NCCL) every rank runs the
same per-GPU batch (weak scaling); logits are gathered to rank 0 over NCCL
once per 16-batch replay.  Rank 0 prints ONE JSON line.

C1/C2 keep several independent batches in flight per GPU (one engine and CUDA
stream each, STREAMS_DEFAULT): a single C2 forward is a latency-bound launch
on a fraction of the SMs, so batches overlap; every batch is still one full
forward, and the timed region covers all K of them.

Timing: W untimed warm-up steps, then exactly K steps bracketed by a barrier
and cudaDeviceSynchronize on both sides, device-timed with CUDA events on the
launching stream, max over ranks.  Inputs rotate over R resident batches whose
total exceeds the 126 MB L2, so each step reads its input from HBM.  Steps are
replayed from CUDA graphs (one graph of R forwards + R single-forward graphs
for the remainder) so host launch overhead stays out of the device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
# independent batches in flight per GPU (one engine + CUDA stream each): the
# C1/C2 forwards are single latency-bound launches that leave SMs idle in their
# split-K reduction tail, so two batches in flight overlap one's tail with the
# other's main loop (measured; bench.py --streams overrides)
STREAMS_DEFAULT = {"c1": 20, "c2": 12}
# K splits per launch (0 = the engine's choice): both run unsplit -- persistent
# CTAs per batch whose epilogue is the straight-line level instantiation, so
# many batches share the GPU without a split-K tail (measured sweep,
# scripts/gpu_splits.sh: C1 split 1 x 20 in flight 4.03 us/batch vs split 2 x 8
# 5.06 us; C2 split 1 x 12 11.15 us vs split 2 14.8 us)
SPLIT_DEFAULT = {"c1": 1, "c2": 1}
PAPER_SAMPLES_PER_S = {  # PAPER.md:603, KANMLP2 G=5 8-bit LUT on RTX 3090
    "c1": 10000 / 5.9e-3, "c2": 10000 / 5.9e-3,
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="wall time of the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=0,
                    help="independent batches in flight (one engine + stream each); 0 = per-config default")
    ap.add_argument("--split-k", type=int, default=0, help="force the K splits of split-K launches")
    return ap.parse_args()


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
                return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


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


def committed_traffic(config: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        v = d.get(config, {}).get("dram_bytes_per_launch")
        return v
    return None


# ---------------------------------------------------------------------------------
def ref_forward(ref, wl, Ws, x, threads):
    """One call of the reference's CPU path on rows x: model_forward for models
    the reference's descriptor schema expresses (bspline-lut mode, per-tensor u8
    W, eval.hpp:70-76, no SiLU term -- the reference has none); for ResKAN18 the
    harness composition of reference functions (oracle/ref_shim.cpp
    ref_graph_forward)."""
    text = json.dumps(wl.descriptor())
    if wl.reference_expressible:
        return ref.model_forward(text, Ws, x, wl.out_size, mode=2, k=wl.lut_k, h=wl.lut_h,
                                 bits_w=8, threads=threads, chunk=256)
    return ref.graph_forward(text, Ws, x, wl.out_size, k=wl.lut_k, h=wl.lut_h, bits_w=8,
                             threads=threads)


def cpu_rows(wl, cores):
    """Rows per reference call: 256-row chunks per thread for the MLPs; for the
    conv models (0.6-9 GOP per sample) one sample per thread."""
    return 2048 if wl.layers is None else cores


def cpu_baseline(wl, seconds: float):
    """The reference's own CPU path (oracle/_ref = the reference headers compiled
    unmodified): model_forward in bspline-lut mode with the reference's weight
    scheme (per-tensor asymmetric u8, eval.hpp:70-76) and no SiLU term (the
    reference has none), batch sharded over all host threads, 256-row chunks.
    Falls back to the C restatement (single thread) if oracle/_ref is absent."""
    from oracle.pyoracle import Oracle, Ref
    Ws, _ = wl.weights()
    cores = os.cpu_count() or 1
    rows = cpu_rows(wl, cores)
    x = wl.inputs(rows, seed=99).astype(np.float64)
    if Ref.available and wl.mode == "spline-table":
        if not wl.reference_expressible:
            raise RuntimeError("spline-table CPU baseline needs a reference-expressible model")
        ref = Ref()
        text = json.dumps(wl.descriptor())
        n, dt = 0, 0.0
        while dt < seconds:
            _, sec = ref.st_model_forward(text, Ws, x, wl.out_size, wl.lut_k, wl.lut_h,
                                          threads=cores, chunk=256)
            n += rows
            dt += sec
        return {"value": n / dt, "unit": "samples/s", "cores": cores, "kind": "reference",
                "sample": f"{n} samples ({rows}-row calls) of {wl.key} through the reference "
                          f"model_forward in spline-table mode (bits_a={wl.lut_k}, h={wl.lut_h}, "
                          f"tables built once, untimed), {cores} threads, {dt:.1f} s"}
    if Ref.available:
        ref = Ref()
        n = 0
        t0 = time.perf_counter()
        while True:
            ref_forward(ref, wl, Ws, x, cores)
            n += rows
            if time.perf_counter() - t0 >= seconds:
                break
        dt = time.perf_counter() - t0
        how = ("model_forward" if wl.reference_expressible else
               "convkan_forward/kan_linear_forward composition (ref_graph_forward)")
        return {"value": n / dt, "unit": "samples/s", "cores": cores, "kind": "reference",
                "sample": f"{n} samples ({rows}-row calls) of {wl.key} through the reference "
                          f"{how} (bspline-lut k{wl.lut_k} h{wl.lut_h}, per-tensor u8 W, no SiLU "
                          f"term), {cores} threads, {dt:.1f} s"}
    o = Oracle()
    g = o.grid(wl.G, wl.P)
    n = 0
    t0 = time.perf_counter()
    if wl.layers is not None:
        raise RuntimeError("oracle/_ref not built: no CPU baseline for conv models")
    while time.perf_counter() - t0 < seconds:
        h = x[:256]
        for w in Ws:
            h = o.lut_forward(g, wl.lut_k, wl.lut_h, 8, h, w)
        n += 256
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "samples/s", "cores": 1, "kind": "port",
            "sample": f"{n} samples of {wl.key} through the C restatement, 1 thread, {dt:.1f} s"}


def run_reference(args):
    """--impl reference: the reference's CPU implementation on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2603_17230_b200 import configs
    from oracle.pyoracle import Ref
    wl = configs.get(args.config)
    cores = os.cpu_count() or 1
    # MLPs: one >=256-row chunk per thread; conv models: one sample per thread
    rows = 256 * cores if wl.layers is None else cores
    x = wl.inputs(rows, seed=7).astype(np.float64)
    Ws, _ = wl.weights()
    if not Ref.available:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    ref = Ref()

    st_mode = wl.mode == "spline-table"
    if st_mode:  # tables built once per call outside the timed forwards
        if not wl.reference_expressible:
            print(json.dumps({"impl": "reference", "unavailable": "the reference's model_forward "
                              "cannot run this model in spline-table mode"}))
            return
        text = json.dumps(wl.descriptor())

    def step():
        if st_mode:
            return ref.st_model_forward(text, Ws, x, wl.out_size, wl.lut_k, wl.lut_h,
                                        threads=cores, chunk=256)[1]
        t = time.perf_counter()
        ref_forward(ref, wl, Ws, x, cores)
        return time.perf_counter() - t
    t_step = step()  # first warm-up step also sizes the run (whole run within ~2 minutes)
    steps = max(1, min(args.steps, 50, int(120.0 / max(t_step, 1e-3))))
    for _ in range(min(args.warmup, 3) - 1):
        step()
    dt = 0.0
    for _ in range(steps):
        dt += step()
    v = rows * steps / dt
    print(json.dumps({
        "impl": "reference",
        "metric": "KAN samples/sec (spline-table path)" if st_mode else "KAN samples/sec (int8-LUT path)",
        "value": v,
        "unit": "samples/s", "n_gpus": args.gpus, "steps": steps, "warmup": min(args.warmup, 3),
        "ms_per_step": dt / steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.key + ": " + wl.title, "batch_per_step": rows,
                   "note": "reference CPU path: " + (
                       f"model_forward in spline-table mode, bits_a={wl.lut_k} h={wl.lut_h}, "
                       "tables built once outside the timed forwards" if st_mode else (
                           ("model_forward" if wl.reference_expressible else
                            "composition of convkan_forward / kan_linear_forward (ref_graph_forward)")
                           + f" bspline-lut k{wl.lut_k} h{wl.lut_h}, per-tensor u8 W, no SiLU"))},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": f"{steps} steps x {rows} rows, {cores} threads"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": f"--steps capped at {steps} so the CPU run stays within about two minutes",
    }))


# ---------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2603_17230_b200 import Engine, EvalOptions, OUT_I8, OUT_F32, W_PER_CHANNEL_SYM
    from paper_2603_17230_b200 import configs
    from paper_2603_17230_b200.sharding import gather_logits

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    wl = configs.get(args.config)
    B = wl.batch  # per-GPU batch (weak scaling)

    Ws, Bs = wl.weights()
    n_streams = args.streams or STREAMS_DEFAULT.get(wl.key, 1)
    engines = []
    for _ in range(n_streams):  # one engine per stream: independent workspaces
        e_ = Engine(wl.descriptor(), local)
        for i, (w, b) in enumerate(zip(Ws, Bs)):
            e_.set_coeffs(i, w, b)
        engines.append(e_)
    eng = engines[0]
    opts = EvalOptions(mode=wl.mode, lut_k=wl.lut_k, lut_h=wl.lut_h, bits_w=wl.bits_w,
                       w_scheme=W_PER_CHANNEL_SYM, silu_base=wl.silu, out_kind=OUT_F32,
                       split_k=args.split_k or SPLIT_DEFAULT.get(wl.key, 0))
    for e_ in engines:
        e_.configure(opts)

    # rotating resident input batches, total > L2
    in_bytes = B * wl.input_size * 4
    R = max(2, min(64, math.ceil(2 * L2_BYTES / in_bytes)))
    R = max(R, 16) if in_bytes < 64 * 1024 * 1024 else R
    xs = [torch.from_numpy(wl.inputs(B, seed=100 * rank + r)).to(dev) for r in range(R)]
    if wl.int8_out:
        y = eng.model_forward(xs[0]).float()
        s_out = float(y.abs().max().item()) / 127.0
        opts.out_kind, opts.out_scale = OUT_I8, s_out
        for e_ in engines:
            e_.configure(opts)
    out_dtype = torch.int8 if wl.int8_out else torch.float32
    outs = torch.empty((R, B, wl.out_size), device=dev, dtype=out_dtype)
    st = torch.cuda.Stream(dev)
    aux = [torch.cuda.Stream(dev) for _ in range(n_streams - 1)]
    streams = [st] + aux
    torch.cuda.synchronize()
    # warm the engines (allocations happen outside graph capture)
    for k, e_ in enumerate(engines):
        with torch.cuda.stream(streams[k]):
            for r in range(R):
                e_.model_forward(xs[r], out=outs[r], stream=streams[k])
    torch.cuda.synchronize()
    launches_per_step = eng.last_launches

    # the R-forward graph: batch r runs on stream r % n_streams (its own engine),
    # forked from and joined back into the capture stream
    big = torch.cuda.CUDAGraph()
    with torch.cuda.graph(big, stream=st):
        for s_ in aux:
            s_.wait_stream(st)
        for r in range(R):
            k = r % n_streams
            engines[k].model_forward(xs[r], out=outs[r], stream=streams[k])
        for s_ in aux:
            st.wait_stream(s_)
    singles = []
    for r in range(R):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            eng.model_forward(xs[r], out=outs[r], stream=st)
        singles.append(g)
    gathered = []

    def run_steps(n):
        q, rem = divmod(n, R)
        for _ in range(q):
            big.replay()
            if world > 1:
                gathered.append(gather_logits(outs.view(R * B, -1), R * B * world))
        for r in range(rem):
            singles[r].replay()

    with torch.cuda.stream(st):
        run_steps(args.warmup)
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
        run_steps(args.steps)
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
    value = world * B * args.steps / (ms / 1e3)

    # ---- dominant kernel: per-launch device time with CUDA events (engine profiling)
    # (the event pairs are recorded as graph nodes around each kernel node, so
    # host launch gaps stay out of the per-launch device time)
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
    lut = wl.mode == "bspline-lut"
    st_mode = wl.mode == "spline-table"
    peaks, peak_src = measured_peaks()
    # bound of the dominant (largest-time) layer
    dom = int(np.argmax(layer_ms))
    bytes_l = wl.layer_bytes_per_launch(dom, B)
    ops_l = wl.layer_ops_per_launch(dom, B)
    whole = launches_per_step == 1 or n_streams > 1
    if whole:
        # the whole forward is one launch (fused output layer), or several
        # batches are in flight (per-launch event brackets cannot isolate one
        # launch): model input in, model output out, every layer's weights
        # once per batch, over the effective time per batch
        bytes_l = (B * wl.input_size * 4 + B * wl.out_size * (1 if wl.int8_out else 4)
                   + sum(wl.weight_bytes(li) for li in range(wl.n_kan)))
        ops_l = wl.ops_per_sample() * B
    int8_peak_tops = peaks.get("int8_tops", 4500.0)
    if lut and "int8_tops" not in peaks and ops_l / bytes_l > 4500e12 / (peaks["hbm_gbs"] * 1e9):
        meas = measure_int8_peak(dev)
        if meas:
            peaks["int8_tops"] = int8_peak_tops = meas
    # a step that is a single launch (C1/C2: the output layer runs fused):
    # the kernel's live average over the timed region is the step time (the
    # profiling pass's event nodes would break the overlap between steps)
    if whole:
        layer_ms[dom] = ms / args.steps
    t_l = layer_ms[dom] / 1e3
    ai = ops_l / bytes_l
    tensor_peak = int8_peak_tops * 1e12 if lut else peaks.get("bf16_tflops", 1677.7) * 1e12
    hbm_peak = peaks["hbm_gbs"] * 1e9
    if st_mode or ai < tensor_peak / hbm_peak:  # spline tables: gather + integer add, no tensor work
        roof = {"bound": "hbm", "achieved": bytes_l / t_l / 1e9, "peak": peaks["hbm_gbs"],
                "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": ops_l / t_l / 1e12,
                "peak": tensor_peak / 1e12, "unit": "TOP/s" if lut else "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = committed_traffic(wl.key)
    kl = wl.kan_layers()[dom]
    roof["kernel"] = (("kan_st_layer" if st_mode else "kan_gather_gemm")
                      + f" KAN layer {dom} ({kl['n_in']}->{kl['n_out']}"
                      + (f", {kl['pix']} px/sample)" if kl["pix"] > 1 else ")"))
    if launches_per_step == 1 and wl.n_kan > 1:
        roof["kernel"] += f" with the {wl.n_kan - 1} following layer(s) fused in"
    if n_streams > 1:
        roof["kernel"] = (f"whole forward ({launches_per_step} launch(es) per batch, "
                          f"{n_streams} batches in flight)")
    roof["per_launch"] = {"algorithmic_bytes": bytes_l, "algorithmic_ops": ops_l,
                          "avg_ms": layer_ms[dom], "launches_timed": prof_steps,
                          "timing": (f"timed region / steps ({n_streams} batches in flight)" if n_streams > 1
                                     else "timed region / steps (one launch per step)" if launches_per_step == 1
                                     else "CUDA event pair around the kernel node, graph replay")}
    roof["peak_source"] = peak_src + (
        "" if not lut or "int8_tops" in peaks else "; int8 peak = datasheet 4.5 POPS dense")
    roof["layer_avg_ms"] = layer_ms
    roof["share_of_step"] = layer_ms[dom] / (ms / args.steps)

    # ---- e2e through the public API: host buffers, H2D + forward + D2H every step
    # (two host threads each drive their own engine and stream, so one call's
    # host->device copy overlaps the other's forward; the C ABI call releases
    # the GIL)
    e2e_steps = max(10, min(args.steps, 300))
    n_e2e = 2
    e2e_steps -= e2e_steps % n_e2e
    e2e_engines, e2e_streams = list(engines[:n_e2e]), list(streams[:n_e2e])
    while len(e2e_engines) < n_e2e:  # a second engine / stream for the overlap
        e_ = Engine(wl.descriptor(), local)
        for i, (w, b) in enumerate(zip(Ws, Bs)):
            e_.set_coeffs(i, w, b)
        e_.configure(opts)
        e2e_engines.append(e_)
        e2e_streams.append(torch.cuda.Stream(dev))
    hx = [torch.from_numpy(wl.inputs(B, seed=500 + r)).pin_memory() for r in range(4)]
    houts = [torch.empty((B, wl.out_size), dtype=out_dtype).pin_memory() for _ in range(n_e2e)]

    def e2e_worker(k, n):
        for i in range(n):
            e2e_engines[k].forward_host_ptr(hx[(i + k) % 4].data_ptr(), B, houts[k].data_ptr(),
                                            stream=e2e_streams[k])
    for k in range(n_e2e):
        e2e_worker(k, 3)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    ths = [threading.Thread(target=e2e_worker, args=(k, e2e_steps // n_e2e)) for k in range(n_e2e)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": world * B * e2e_steps / e2e_s, "unit": "samples/s",
           "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": B * wl.out_size *
           (1 if wl.int8_out else 4), "steps": e2e_steps,
           "api": "kan_engine_forward_host (pinned host buffers, stream-synchronous)",
           "host_threads": n_e2e}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(wl, args.cpu_seconds)
        except Exception as ex:  # report, never hide
            cpu = {"value": None, "error": str(ex)}

    if rank == 0:
        paper = PAPER_SAMPLES_PER_S.get(wl.key)
        line = {
            "metric": "KAN samples/sec (int8-LUT path)" if lut else f"KAN samples/sec ({wl.mode} path)",
            # spline-table lines: roofline.per_launch.algorithmic_ops counts table
            # lookups + integer adds (one per connection), not multiply-adds
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": (value / paper) if paper else None,
            "dtype": "u8" if (lut or st_mode) else wl.mode, "data": "synthetic",
            "config": {"workload": wl.key + ": " + wl.title, "batch_per_gpu": B,
                       "global_batch": B * world, "parallelism": f"dp{world}",
                       "l2": f"inputs rotate over {R} resident batches "
                             f"({R * in_bytes / 2**20:.0f} MiB > 126 MiB L2)",
                       "launch": f"CUDA graphs ({R}-forward graph + single-forward graphs)",
                       "streams": n_streams,
                       "split_k": opts.split_k or "auto",
                       "concurrency": (f"{n_streams} independent batches in flight (one engine + CUDA "
                                       "stream each); ms_per_step = timed region / steps"
                                       if n_streams > 1 else "one batch at a time"),
                       "vs_baseline_ref": "PAPER.md:603 KANMLP2 G=5 8-bit LUT, RTX 3090, "
                                          "1.69M samples/s" if paper else None},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(t_wall0, t_wall1),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the Walsh->wavelet change-of-basis hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

metric : forward+adjoint matvecs/s (a matvec = one U W^-1 or one W U* application
         to one vector/image) and the achieved fraction of the HBM roofline.
step   : config 1-4: one forward of the whole batch + one adjoint of the whole
         batch (2*batch matvecs; independent, so on two streams); config 5: 50
         iterations of the normal operator U*U on the image (100 matvecs).
         Default config: 2 (BASELINE configs[1]).  The step is captured once into
         a CUDA graph per rank and replayed (same launches, no per-launch host
         overhead; eager fallback if capture or a bitwise replay check fails;
         config 5 on P > 1 GPUs, whose step holds NCCL all-to-alls, stays eager).
value  : whole-job throughput, inputs resident in HBM, device-timed with CUDA
         events per step, L2 flushed (256 MiB write) between steps, max over ranks.
e2e    : the same metric through the public API with the step's inputs copied
         from pinned host memory and the results copied back, inside the timed
         region.
roofline: dominant kernel (largest device time), algorithmic bytes
          / its CUDA-event time, vs MEASURED_PEAKS.json.
cpu_baseline: the reference library itself (oracle/_ref, built from
         /root/reference) on the host cores, rank 0 at N = 1, bounded sample.
Multi-GPU: one process per GPU (torchrun); independent batches per rank,
         no data-path collective ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# (family, nu, boundary, j, q, dim, r0, batch, input kind, density, workload name)
CONFIGS = {
    1: (0, 1, 0, 10, 1, 1, 1, 1, 0, 1.0, "cfg1: 1D Haar r0=1 M=2^10 q=1, single vector"),
    2: (0, 4, 1, 16, 2, 1, 4, 64, 1, 1.0, "cfg2: 1D db4 boundary-VMP r0=4 M=2^16 q=2 (N=2^18), batch 64, level-decaying coeffs"),
    3: (0, 3, 1, 21, 2, 1, 4, 32, 0, 0.1, "cfg3: 1D db3 boundary-VMP r0=4 M=2^21 q=2 (N=2^23), batch 32, 10% nonzeros"),
    4: (0, 4, 1, 10, 1, 2, 4, 16, 1, 0.05, "cfg4: 2D db4 boundary-VMP r0=4 M=1024^2 q=1 (N=2048^2), batch 16, 5% nonzeros"),
    5: (0, 2, 1, 12, 1, 2, 3, 1, 0, 0.02, "cfg5: 2D db2 boundary-VMP r0=3 M=4096^2 q=1 (N=8192^2), 50 U*U iterations, 2% nonzeros"),
}
CFG5_ITERS = 50


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(cfg, kernel: str, batch: int) -> float:
    """Minimal DRAM bytes of one step's launches of `kernel`."""
    fam, nu, bnd, j, q, dim, r0 = cfg[:7]
    M, N = 1 << j, 1 << (j + q)
    if kernel in ("normal_rows", "transpose"):
        # banded normal form (config 5): every launch reads and writes each
        # M-row once; per U*U: 2 row passes + 1 transpose over the M x M image
        per_iter = 2 if kernel == "normal_rows" else 1
        iters = CFG5_ITERS if cfg is CONFIGS[5] else 1
        return 16.0 * batch * (M * M if dim == 2 else M) * per_iter * iters
    if dim == 2:
        mats = CFG5_ITERS if cfg is CONFIGS[5] else 1
        # small_fwd: row pass (M^2 -> MN) + column pass (MN -> N^2); small_adj mirrored
        return 8.0 * batch * mats * (M * M + 2 * M * N + N * N)
    CW = 32 + 2 * (nu - 1)
    A = M // 32
    lc = min(j - 1, 10)  # coarse levels <= 10 run in k_wav_coarse / the analysis tail (CWW_PYR_SYN_BOT)
    per = {
        "small_fwd": M + N, "small_adj": M + N,
        "large_fwd1": M + A * CW, "large_fwd1_syn": M + A * CW, "large_fwd2": A * CW + N,
        "large_adj2": N + A * CW, "large_adj1": A * CW + M,
        # all launches of a step together: every coefficient read once, every sample written once
        "idwt_pyr": 2 * M, "dwt_pyr": 2 * M,
        "wav_coarse": 2 * (1 << lc),
    }
    return 8.0 * batch * per.get(kernel, 0)


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU implementation, all host threads."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import numpy as np
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = cfg
    threads = os.cpu_count() or 1
    kind_s = "reference"
    try:
        from oracle_py import Reference
        R = Reference()
        op = R.op(fam, nu, bnd, j, q, dim, r0)
    except Exception as e:  # noqa: BLE001 -- reference not built: the C restatement
        from oracle_py import Oracle
        kind_s = "port"
        op = None
        err = str(e)
    # bounded sample per step: config 1-4 up to `threads` vectors/images, config 5: 1 iteration
    if cfg is CONFIGS[5]:
        sample, iters, matv = 1, 1, 2
    else:
        sample = min(batch, max(1, threads)) if dim == 1 else 1
        iters, matv = 1, 2 * sample
    from paper_2106_00554_b200 import synth  # input generator only (host, no GPU)
    M, N = 1 << j, 1 << (j + q)
    nin, nout = (M, N) if dim == 1 else (M * M, N * N)
    xs = np.stack([synth(kind, 1000 * args.config + b, j, r0, dens, dim) for b in range(sample)])
    rng = np.random.default_rng(args.config)
    ys = rng.standard_normal((sample, nout))
    outf = np.empty((sample, nout))
    outa = np.empty((sample, nin))

    def one_step():
        if op is None:
            raise RuntimeError("reference library unavailable: " + err)
        if cfg is CONFIGS[5]:
            t = op.bench(2, xs, outa, 1, threads, iters)
        else:
            t = op.bench(0, xs, outf, sample, threads)
            t += op.bench(1, ys, outa, sample, threads)
        return t

    for _ in range(args.warmup):
        one_step()
    ts = [one_step() for _ in range(args.steps)]
    total = sum(ts)
    value = matv * args.steps / total
    line = {
        "impl": "reference", "metric": "forward+adjoint matvecs/s", "value": value, "unit": "matvec/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded test_rng inputs, SURVEY.md 8d)",
        "config": {"workload": name, "batch": batch, "sample_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": threads, "kind": kind_s,
                         "sample": f"{sample} vector(s) forward + adjoint per step" if cfg is not CONFIGS[5]
                         else "1 U*U iteration per step (of the 50-iteration config)"},
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline(cfg, config_id):
    """Reference CPU path on a bounded sample (rank 0, N = 1)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import numpy as np
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = cfg
    threads = os.cpu_count() or 1
    try:
        from oracle_py import Reference
        op = Reference().op(fam, nu, bnd, j, q, dim, r0)
        kind_s = "reference"
    except Exception:  # noqa: BLE001
        from oracle_py import Oracle
        op = None
        kind_s = "port"
    from paper_2106_00554_b200 import synth
    M, N = 1 << j, 1 << (j + q)
    nin, nout = (M, N) if dim == 1 else (M * M, N * N)
    if cfg is CONFIGS[5]:
        sample = 1
    else:
        sample = min(batch, threads) if dim == 1 else 1
    xs = np.stack([synth(kind, 1000 * config_id + b, j, r0, dens, dim) for b in range(sample)])
    ys = np.random.default_rng(0).standard_normal((sample, nout))
    outf, outa = np.empty((sample, nout)), np.empty((sample, nin))
    if op is None:
        from oracle_py import Oracle
        o = Oracle().op(fam, nu, bnd, j, q, dim, r0)
        t0 = time.perf_counter()
        for b in range(sample):
            o.forward(xs[b])
            o.adjoint(ys[b])
        t = time.perf_counter() - t0
        return {"value": 2 * sample / t, "unit": "matvec/s", "cores": 1, "kind": "port",
                "sample": f"{sample} vector(s) forward + adjoint"}
    total, mv, reps = 0.0, 0, 0
    while total < 8.0 and reps < 50:
        if cfg is CONFIGS[5]:
            total += op.bench(2, xs, outa, 1, threads, 1)
            mv += 2
        else:
            total += op.bench(0, xs, outf, sample, threads) + op.bench(1, ys, outa, sample, threads)
            mv += 2 * sample
        reps += 1
    return {"value": mv / total, "unit": "matvec/s", "cores": threads, "kind": kind_s,
            "sample": (f"{reps} x ({sample} vector(s) forward + adjoint), one std::thread per vector"
                       if cfg is not CONFIGS[5] else f"{reps} U*U iteration(s), FastOp::set_threads({threads})"),
            "seconds": total}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = cfg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg)
        return

    import numpy as np
    import torch
    import paper_2106_00554_b200 as cw

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    is5 = args.config == 5
    rowpart = is5 and world > 1  # config 5 on P GPUs: rows partitioned, all-to-all transposes
    if nu == 1:
        op = cw.HaarFullRankOp(j, q, r0)
    elif rowpart:
        from paper_2106_00554_b200.dist import RowPartitioned2D, cuda_apply_1d, cuda_normal_1d
        op1 = cw.ComposedOp(cw.FastOp(spec, j, q, 1), None, True, r0)
        d2 = RowPartitioned2D(1 << j, 1 << (j + q), cuda_apply_1d(op1), apply_normal_1d=cuda_normal_1d(op1))
        op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
    else:
        op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
    nin, nout = op.cols(), op.rows()
    # per-rank inputs (weak scaling: each rank owns a full batch)
    xs = np.stack([cw.synth(kind, 1000 * args.config + rank * batch + b, j, r0, dens, dim)
                   for b in range(batch)])
    g = torch.Generator(device="cpu").manual_seed(1000 * args.config + 500 + rank)
    ys = torch.randn((batch, nout), generator=g, dtype=torch.float64)
    x_pin = torch.from_numpy(xs).pin_memory()
    y_pin = ys.pin_memory()
    x_dev, y_dev = x_pin.to(dev), y_pin.to(dev)
    fo_dev = torch.empty((batch, nout), dtype=torch.float64, device=dev)
    ao_dev = torch.empty((batch, nin), dtype=torch.float64, device=dev)
    fo_pin = torch.empty((batch, nout), dtype=torch.float64).pin_memory()
    ao_pin = torch.empty((batch, nin), dtype=torch.float64).pin_memory()
    flush = torch.empty(256 << 20 >> 3, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    mv_per_step = 2 * CFG5_ITERS if is5 else 2 * batch
    if rowpart:
        M_ = 1 << j
        mr = M_ // world
        x_rows0 = x_dev.view(M_, M_)[rank * mr:(rank + 1) * mr].contiguous()

    # forward and adjoint of the step are independent: two streams, so one chain's
    # latency-bound launches overlap the other's (inside the replayed CUDA graph:
    # cfg2 0.210 vs 0.240 ms sequential; eager launches measured no gain)
    conc = os.environ.get("CWW_BENCH_CONCURRENT", "1") == "1"
    # stream priorities (env CWW_BENCH_PRIO = f,a; lower = higher priority): the
    # adjoint chain is the longer one, so it goes first and the forward fills the
    # gaps (cfg2 0.1985 vs 0.2024 ms; the forward first: 0.225 ms)
    pf, pa = (int(t) for t in os.environ.get("CWW_BENCH_PRIO", "0,-1").split(","))
    s_dev_f, s_dev_a = torch.cuda.Stream(dev, priority=pf), torch.cuda.Stream(dev, priority=pa)

    def step_device(concurrent=conc):
        if rowpart:
            d2.normal(x_rows0, CFG5_ITERS)
        elif is5:
            ao_dev.copy_(x_dev)
            op.normal(ao_dev, iters=CFG5_ITERS, work=fo_dev)
        elif concurrent:
            # forward and adjoint of the batch are independent: two streams, so one
            # chain's latency-bound phases and launch tails overlap the other's
            cur = torch.cuda.current_stream(dev)  # (the capture stream inside a graph capture)
            s_dev_f.wait_stream(cur)
            s_dev_a.wait_stream(cur)
            with torch.cuda.stream(s_dev_f):
                op.forward(x_dev, fo_dev)
            with torch.cuda.stream(s_dev_a):
                op.adjoint(y_dev, ao_dev)
            cur.wait_stream(s_dev_f)
            cur.wait_stream(s_dev_a)
        else:
            op.forward(x_dev, fo_dev)
            op.adjoint(y_dev, ao_dev)

    s_fwd, s_adj = torch.cuda.Stream(dev, priority=pf), torch.cuda.Stream(dev, priority=pa)

    def step_e2e():
        if not (rowpart or is5):
            # the public host API on pinned buffers (cww_*_host_async): chunk-pipelined H2D /
            # compute / D2H; forward and adjoint are independent, so they run on two streams
            # and the two PCIe directions overlap.  Tiny inputs (config 1) go zero-copy: the
            # kernels read and write the pinned buffers over PCIe, no copy launches.
            cur = torch.cuda.current_stream(dev)  # (the capture stream inside a graph capture)
            s_fwd.wait_stream(cur)
            s_adj.wait_stream(cur)
            with torch.cuda.stream(s_fwd):
                op.forward(x_pin, fo_pin)
            with torch.cuda.stream(s_adj):
                op.adjoint(y_pin, ao_pin)
            cur.wait_stream(s_fwd)
            cur.wait_stream(s_adj)
            return
        x_dev.copy_(x_pin, non_blocking=True)
        if rowpart:
            xr = d2.normal(x_dev.view(1 << j, 1 << j)[rank * mr:(rank + 1) * mr], CFG5_ITERS)
            ao_pin.view(1 << j, 1 << j)[rank * mr:(rank + 1) * mr].copy_(xr, non_blocking=True)
        elif is5:
            ao_dev.copy_(x_dev)
            op.normal(ao_dev, iters=CFG5_ITERS, work=fo_dev)
            ao_pin.copy_(ao_dev, non_blocking=True)
        else:
            y_dev.copy_(y_pin, non_blocking=True)
            op.forward(x_dev, fo_dev)
            op.adjoint(y_dev, ao_dev)
            fo_pin.copy_(fo_dev, non_blocking=True)
            ao_pin.copy_(ao_dev, non_blocking=True)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier()
        torch.cuda.synchronize(dev)
        for a, b in evs:
            flush.zero_()  # evict L2 between steps (outside the event pair)
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def graphed(fn, outs):
        """The step captured once into a CUDA graph and replayed (the launch-bound
        configs lose their per-launch host overhead); falls back to eager calls
        when capture fails or a replay does not reproduce the eager outputs bit
        for bit.  Returns (callable, kernel launches per step or None)."""
        if os.environ.get("CWW_BENCH_GRAPH", "1") != "1":
            return fn, None
        try:
            fn()
            torch.cuda.synchronize(dev)
            ref = [o.clone() for o in outs]
            g = torch.cuda.CUDAGraph()
            l0 = cw.kernel_launches()
            with torch.cuda.graph(g):
                fn()
            per = cw.kernel_launches() - l0
            for o in outs:
                o.zero_()
            g.replay()
            torch.cuda.synchronize(dev)
            if all(torch.equal(o, r) for o, r in zip(outs, ref)):
                return g.replay, per
        except Exception as e:  # noqa: BLE001 -- any capture problem: eager calls
            print(f"bench: CUDA graph capture not used ({type(e).__name__}: {e})", file=sys.stderr)
        torch.cuda.synchronize(dev)
        return fn, None

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize(dev)
    dev_outs = [ao_dev] if (is5 or rowpart) else [fo_dev, ao_dev]
    step_dev_g, per_launch = graphed(step_device, dev_outs) if not rowpart else (step_device, None)
    for _ in range(args.warmup):
        step_dev_g()
    torch.cuda.synchronize(dev)

    l0 = cw.kernel_launches()
    with Clocks(local) as clk:
        ms = timed(step_dev_g, args.steps)  # the reported time: no per-launch instrumentation
        launches = cw.kernel_launches() - l0 if per_launch is None else per_launch * args.steps
        # per-kernel breakdown: the same steps again with CUDA events around every launch
        cw.profile_enable(True)
        cw.profile_dump()
        ms_prof = timed(lambda: step_device(False), args.steps)  # sequential: clean per-kernel events
        cw.profile_enable(False)
        prof = cw.profile_dump()
        t_end = time.time() + 1.0  # keep the same load running so nvidia-smi sees it
        while time.time() < t_end:
            step_device()
            torch.cuda.synchronize(dev)

    for _ in range(2):
        step_e2e()
    e2e_outs = [ao_pin] if (is5 or rowpart) else [fo_pin, ao_pin]
    step_e2e_g, _ = graphed(step_e2e, e2e_outs) if not rowpart else (step_e2e, None)
    for _ in range(2):
        step_e2e_g()
    ms_e2e = timed(step_e2e_g, args.steps)

    # weak scaling (independent batches per rank) except config 5 on P GPUs,
    # where the one image is shared (strong scaling)
    total_mv = mv_per_step * args.steps * (1 if rowpart else world)
    value = total_mv / (ms / 1e3)
    e2e = total_mv / (ms_e2e / 1e3)
    h2d = x_pin.numel() * 8 + (0 if is5 else y_pin.numel() * 8)
    d2h = ao_pin.numel() * 8 + (0 if is5 else fo_pin.numel() * 8)

    # roofline of the dominant kernel
    peak, peak_kind = peaks()
    roof = None
    if prof:
        kname = max(prof, key=lambda k: prof[k][0])
        kms, kn = prof[kname]
        steps_bytes = algorithmic_bytes(cfg, kname, batch) * args.steps
        achieved = steps_bytes / (kms / 1e3) / 1e9 if kms > 0 else 0.0
        traffic, tnote = None, None
        try:  # committed ncu captures of this config's leading kernels (profiles/r01_traffic.json)
            trs = json.load(open(os.path.join(REPO, "profiles", "r01_traffic.json")))[str(args.config)]
            for tr in (trs if isinstance(trs, list) else [trs]):
                if tr["kernel"] == kname:
                    traffic, tnote = tr["bytes"], tr["launch"] + " (ncu dram__bytes_read+write, profiles/)"
        except (OSError, KeyError, ValueError):
            pass
        roof = {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_launch": tnote, "kernel_ms_per_launch": kms / kn, "launches": kn,
                "kernel_share_of_step": round(kms / ms_prof, 4)}
    M, N = 1 << j, 1 << (j + q)
    per_mv = 8 * ((M + N) if dim == 1 else (M * M + N * N))
    path_gbs = per_mv * total_mv / world / (ms / 1e3) / 1e9

    line = {
        "metric": "forward+adjoint matvecs/s", "value": round(value, 3), "unit": "matvec/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if rowpart else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded test_rng inputs, SURVEY.md 8d)",
        "config": {"workload": name, "batch_per_gpu": batch,
                   "step": (f"{CFG5_ITERS} x U*U on the image (cww_normal: banded normal form W G W^-1 per "
                            "axis, G = U*U exactly banded since H^T H = M I; rows fused IDWT-band-DWT, tiled "
                            "transposes)" if is5 else
                            ("forward + adjoint of the batch (independent: two streams)" if conc else
                             "forward + adjoint of the batch")),
                   "launch": ("one CUDA graph per step (captured once, replayed; eager fallback)"
                              if per_launch is not None else "eager launches"),
                   "l2": "flushed (256 MiB write) between timed steps",
                   "parallelism": (f"rows/{world} + NCCL all-to-all transposes" if rowpart
                                   else f"dp{world} (independent batches)")},
        "path_gbs_per_gpu": round(path_gbs, 1), "path_frac": round(path_gbs / peak, 4),
        **({"path_frac_kind": "effective (algorithmic bytes 2*8(M^2+N^2) per U*U; the banded normal form "
                              "moves 3*16*M^2 per U*U on one GPU)",
            "actual_hbm_frac": round(3 * 16 * (1 << j) ** 2 * CFG5_ITERS * args.steps
                                     / (ms / 1e3) / 1e9 / peak, 4)} if is5 and not rowpart else {}),
        "roofline": roof,
        "kernels": {k: [round(v[0] / args.steps, 4), v[1] // args.steps] for k, v in prof.items()},
        "gpu_launches": launches,
        "e2e": {"value": round(e2e, 3), "unit": "matvec/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e / args.steps, 4),
                # host link throughput of the e2e step (PCIe Gen5 x16 on this box: ~55 GB/s per
                # direction, ~99 GB/s both directions at once, tools/pcie_bw.py)
                "link_gbs": round((h2d + d2h) / (ms_e2e / args.steps / 1e3) / 1e9, 1)},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args.config)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

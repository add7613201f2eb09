#!/usr/bin/env python
"""Benchmark of the Walsh->wavelet change-of-basis hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

metric : forward+adjoint matvecs/s (a matvec = one U W^-1 or one W U* application
         to one vector/image) and the achieved fraction of the HBM roofline.
step   : config 1-4: one forward of the whole batch + one adjoint of the whole
         batch (2*batch matvecs; independent, so on two streams); config 5: 50
         iterations of the normal operator U*U on the image (100 matvecs).
         Default config: 3 (M = 2^21, N = 2^23, batch 32: the north_star's
         2^23-length target and the largest 1D configuration).  The step is
         captured once into a CUDA graph per rank and replayed (eager fallback if
         capture or a bitwise replay check fails).
inputs : seeded synthetic data of SURVEY.md 8d (test_rng): vector b of config c
         has seed 1000c + b (forward input) and 1000c + 500 + b (adjoint input,
         N(0,1)); the same generator and seeds feed --impl reference.
value  : whole-job throughput, inputs resident in HBM, device-timed with CUDA
         events per step, L2 flushed (256 MiB write) between steps, max over ranks.
e2e    : the same metric through the public API with the step's inputs copied
         from pinned host memory and the results copied back, inside the timed
         region.
roofline: dominant kernel (largest device time); its algorithmic bytes are its
         share of the path's SURVEY 8(d) bytes (8(M+N) per 1D matvec, 8(M^2+N^2)
         per 2D matvec): only the path's own inputs and outputs it reads or
         writes, intermediates excluded.  Peak from MEASURED_PEAKS.json.
cpu_baseline: the reference library itself (oracle/_ref, built from
         /root/reference) on the host cores, rank 0 at N = 1, bounded sample.
Multi-GPU: one process per GPU (torchrun).  Configs 2-4: the fixed global batch
         is sharded across ranks (dist.shard_batch, no data-path collective,
         "scaling": "strong" -- the total work is fixed).  Config 1: independent
         replicas ("weak").  Config 5: rows partitioned, NCCL all-to-all
         transposes through the C ABI (cww_dist_*, "strong").
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# (family, nu, boundary, j, q, dim, r0, global batch, input kind, density, workload name)
CONFIGS = {
    1: (0, 1, 0, 10, 1, 1, 1, 1, 0, 1.0, "cfg1: 1D Haar r0=1 M=2^10 q=1, single vector"),
    2: (0, 4, 1, 16, 2, 1, 4, 64, 1, 1.0, "cfg2: 1D db4 boundary-VMP r0=4 M=2^16 q=2 (N=2^18), batch 64, level-decaying coeffs"),
    3: (0, 3, 1, 21, 2, 1, 4, 32, 0, 0.1, "cfg3: 1D db3 boundary-VMP r0=4 M=2^21 q=2 (N=2^23), batch 32, 10% nonzeros"),
    4: (0, 4, 1, 10, 1, 2, 4, 16, 1, 0.05, "cfg4: 2D db4 boundary-VMP r0=4 M=1024^2 q=1 (N=2048^2), batch 16, 5% nonzeros"),
    5: (0, 2, 1, 12, 1, 2, 3, 1, 0, 0.02, "cfg5: 2D db2 boundary-VMP r0=3 M=4096^2 q=1 (N=8192^2), 50 U*U iterations, 2% nonzeros"),
}
DEFAULT_CONFIG = 3
CFG5_ITERS = 50


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def under_profiler() -> bool:
    """ncu / Nsight injection libraries mapped into this process."""
    if os.environ.get("CUDA_INJECTION64_PATH"):
        return True
    try:
        with open("/proc/self/maps") as f:
            return any(("ToolsInjection" in ln) or ("nsight-compute" in ln) or ("InterceptorInjection" in ln)
                       for ln in f)
    except OSError:
        return False


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def shard(config_id: int, world: int, rank: int):
    """(first global item, items on this rank) -- configs 2-4 shard the fixed
    global batch (dist.shard_batch); config 1 runs one replica per rank and
    config 5 has one (row-partitioned) image."""
    cfg = CONFIGS[config_id]
    batch = cfg[7]
    if config_id in (2, 3, 4) and world > 1:
        base, rem = divmod(batch, world)
        return rank * base + min(rank, rem), base + (1 if rank < rem else 0)
    return 0, batch


def scaling_kind(config_id: int, world: int) -> str:
    return "weak" if config_id == 1 else "strong"


def config_dict(config_id: int, world: int) -> dict:
    """The `config` object of the JSON line; identical for both arms."""
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = CONFIGS[config_id]
    if config_id == 5:
        step = (f"{CFG5_ITERS} x U*U on the image (cww_normal: banded normal form W G W^-1 per axis, "
                "G = U*U exactly banded since H^T H = M I)")
        par = f"rows/{world} + all-to-all transposes" if world > 1 else "1 GPU"
    else:
        step = "forward + adjoint of the batch"
        par = (f"{world} independent replicas" if config_id == 1 and world > 1
               else (f"batch sharded {batch}/{world} per GPU (dp{world}, no collective)" if world > 1 else "1 GPU"))
    per = shard(config_id, world, 0)[1]
    return {"workload": name, "global_batch": batch, "batch_per_gpu": per, "step": step,
            "l2": "flushed (256 MiB write) between timed steps", "parallelism": par,
            "inputs": "seeded test_rng (seed 1000c+b; adjoint input 1000c+500+b)"}


def make_inputs(synth, config_id: int, start: int, count: int):
    """Forward inputs (wavelet coefficients) and adjoint inputs (N(0,1) Walsh
    samples) of global items start..start+count-1; `synth` is the product's or
    the oracle's test_rng generator (bit-identical, tests/test_oracle.py)."""
    import numpy as np
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = CONFIGS[config_id]
    xs = np.stack([synth(kind, 1000 * config_id + b, j, r0, dens, dim) for b in range(start, start + count)])
    if config_id == 5:
        return xs, None
    ys = np.stack([synth(0, 1000 * config_id + 500 + b, j + q, r0, 1.0, dim) for b in range(start, start + count)])
    return xs, ys


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


def path_bytes(cfg) -> int:
    """SURVEY 8(d) algorithmic bytes of one matvec: 8(M+N) (1D), 8(M^2+N^2) (2D)."""
    j, q, dim = cfg[3], cfg[4], cfg[5]
    M, N = 1 << j, 1 << (j + q)
    return 8 * ((M + N) if dim == 1 else (M * M + N * N))


def algorithmic_bytes(cfg, kernel: str, nvec: int) -> float:
    """The SURVEY 8(d) bytes that one step's launches of `kernel` account for:
    the path's inputs it reads and the path's outputs it writes (each once);
    intermediates (xi, the Hadamard intermediate G, the 2D row-pass T) are
    excluded.  nvec = vectors (1D) / images (2D) of the step per direction."""
    fam, nu, bnd, j, q, dim, r0 = cfg[:7]
    M, N = 1 << j, 1 << (j + q)
    if kernel in ("normal_rows", "transpose"):
        # banded normal form (config 5): no Walsh-domain output exists; every
        # launch reads and writes the M x M image once (actual bytes, labelled)
        per_iter = 2 if kernel == "normal_rows" else 1
        iters = CFG5_ITERS if cfg is CONFIGS[5] else 1
        return 16.0 * nvec * M * M * per_iter * iters
    if dim == 2:
        # small_fwd: row pass reads X (M^2), column pass writes Y (N^2); small_adj mirrored
        return 8.0 * nvec * (M * M + N * N) if kernel in ("small_fwd", "small_adj", "wv_fwd", "wv_adj") else 0.0
    lc = min(j - 1, 10)  # coarse synthesis levels <= 10 run in k_wav_coarse
    idwt = r0 < j
    per = {
        "small_fwd": M + N, "small_adj": M + N, "wv_fwd": M + N, "wv_adj": M + N,
        "wav_coarse": (1 << lc) if idwt else 0,
        "idwt_pyr": M - (1 << lc),               # the detail coefficients above level lc
        "large_fwd1": 0 if idwt else M, "large_fwd": N if idwt else M + N,
        "large_fwd2": N,
        "large_adj2": N, "large_adj": M if not idwt else N,
        "large_adj1": 0 if idwt else M,
        "dwt_pyr": M,                            # every coefficient written once
    }
    return 8.0 * nvec * per.get(kernel, 0)


def latest_traffic(config_id: int):
    """ncu DRAM bytes per launch of this config's kernels from the newest
    committed profiles/rNN_traffic.json that has the config."""
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "r*_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
            ent = d.get(str(config_id))
        except (OSError, ValueError):
            continue
        if ent:
            return (ent if isinstance(ent, list) else [ent]), os.path.basename(path)
    return [], None


def _ref_op(cfg):
    """The compiled reference (oracle/_ref) or, if it was not built, the C port."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    from oracle_py import Oracle, Reference
    fam, nu, bnd, j, q, dim, r0 = cfg[:7]
    try:
        return Reference().op(fam, nu, bnd, j, q, dim, r0), "reference", Oracle()
    except Exception:  # noqa: BLE001 -- reference not built: the C restatement
        return None, "port", Oracle()


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU implementation (oracle/_ref:
    the unmodified proj/src/{walsh,wavelet,kernel,fastop}.cpp) on every host
    thread, on the GPU arm's inputs, config and metric.  The product package
    is never imported here."""
    import numpy as np
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = cfg
    threads = os.cpu_count() or 1
    op, kind_s, orc = _ref_op(cfg)
    world = args.gpus
    xs, ys = make_inputs(orc.synth, args.config, 0, batch)
    M, N = 1 << j, 1 << (j + q)
    nin, nout = (M, N) if dim == 1 else (M * M, N * N)
    outf = np.empty((batch, nout))
    outa = np.empty((batch, nin))
    if op is None:
        oop = orc.op(fam, nu, bnd, j, q, dim, r0)

    def one_step():
        """The whole batch (configs 1-4); config 5: one U*U iteration of the 50."""
        if op is None:  # scalar port, one thread
            t0 = time.perf_counter()
            if args.config == 5:
                oop.adjoint(oop.forward(xs[0]))
            else:
                for b in range(batch):
                    outf[b] = oop.forward(xs[b])
                    outa[b] = oop.adjoint(ys[b])
            return time.perf_counter() - t0
        if args.config == 5:
            return op.bench(2, xs, outa, 1, threads, 1)
        return op.bench(0, xs, outf, batch, threads) + op.bench(1, ys, outa, batch, threads)

    for _ in range(args.warmup):
        one_step()
    ts = [one_step() for _ in range(args.steps)]
    total = sum(ts)
    matv = 2 if args.config == 5 else 2 * batch
    value = matv * args.steps / total
    sample = ("1 U*U iteration (2 matvecs) of the 50 per step; FastOp::set_threads"
              if args.config == 5 else f"the full batch: {batch} x (forward + adjoint) per step, one std::thread per vector"
              if dim == 1 else f"the full batch: {batch} x (forward + adjoint) per step, FastOp::set_threads")
    line = {
        "impl": "reference", "metric": "forward+adjoint matvecs/s", "value": value, "unit": "matvec/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": scaling_kind(args.config, world),
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded test_rng inputs, SURVEY.md 8d)",
        "config": config_dict(args.config, world),
        "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": threads if op is not None else 1,
                         "kind": kind_s, "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline(cfg, config_id, xs, ys):
    """Reference CPU path on a bounded sample of this rank's inputs (rank 0, N = 1)."""
    import numpy as np
    fam, nu, bnd, j, q, dim, r0 = cfg[:7]
    threads = os.cpu_count() or 1
    op, kind_s, orc = _ref_op(cfg)
    M, N = 1 << j, 1 << (j + q)
    nin, nout = (M, N) if dim == 1 else (M * M, N * N)
    sample = 1 if (config_id == 5 or dim == 2) else min(len(xs), threads)
    xs = np.ascontiguousarray(xs[:sample])
    ys = None if ys is None else np.ascontiguousarray(ys[:sample])
    outf, outa = np.empty((sample, nout)), np.empty((sample, nin))
    if op is None:
        o = orc.op(fam, nu, bnd, j, q, dim, r0)
        t0 = time.perf_counter()
        for b in range(sample):
            o.forward(xs[b])
            if ys is not None:
                o.adjoint(ys[b])
        t = time.perf_counter() - t0
        return {"value": (2 if ys is not None else 1) * sample / t, "unit": "matvec/s", "cores": 1,
                "kind": "port", "cpu_model": cpu_model(), "sample": f"{sample} vector(s) forward + adjoint"}
    total, mv, reps = 0.0, 0, 0
    while total < 8.0 and reps < 50:
        if config_id == 5:
            total += op.bench(2, xs, outa, 1, threads, 1)
            mv += 2
        else:
            total += op.bench(0, xs, outf, sample, threads) + op.bench(1, ys, outa, sample, threads)
            mv += 2 * sample
        reps += 1
    return {"value": mv / total, "unit": "matvec/s", "cores": threads, "kind": kind_s, "cpu_model": cpu_model(),
            "sample": (f"{reps} x ({sample} vector(s) forward + adjoint), one std::thread per vector"
                       if config_id != 5 and dim == 1 else
                       f"{reps} x (1 image forward + adjoint), FastOp::set_threads({threads})" if config_id != 5
                       else f"{reps} U*U iteration(s), FastOp::set_threads({threads})"),
            "seconds": total}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    fam, nu, bnd, j, q, dim, r0, gbatch, kind, dens, name = cfg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.gpus = max(args.gpus, world) if world > 1 else args.gpus

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
        # the C ABI's row-partitioned operator: NCCL grouped send/recv transposes
        import torch.distributed as dist
        from paper_2106_00554_b200.dist import NativeRowPartitioned2D, nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        d2 = NativeRowPartitioned2D(spec, j, q, r0, rank=rank, nranks=world, nccl_id=obj[0], device=local)
        op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
    else:
        op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
    nin, nout = op.cols(), op.rows()
    start, batch = shard(args.config, world, rank)
    xs, ys = make_inputs(cw.synth, args.config, start, batch)
    if ys is None:
        ys = np.zeros((batch, nout))
    x_pin = torch.from_numpy(xs).pin_memory()
    y_pin = torch.from_numpy(ys).pin_memory()
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
        x_rows = torch.empty_like(x_rows0)

    # forward and adjoint of the step are independent: two streams, so one chain's
    # latency-bound launches overlap the other's; the adjoint chain (the longer one)
    # at the higher priority
    s_dev_f, s_dev_a = torch.cuda.Stream(dev, priority=0), torch.cuda.Stream(dev, priority=-1)

    def step_device(concurrent=True):
        if rowpart:
            x_rows.copy_(x_rows0)
            d2.normal(x_rows, CFG5_ITERS)  # in place
        elif is5:
            ao_dev.copy_(x_dev)
            op.normal(ao_dev, iters=CFG5_ITERS, work=fo_dev)
        elif concurrent:
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

    s_fwd, s_adj = torch.cuda.Stream(dev, priority=0), torch.cuda.Stream(dev, priority=-1)

    def step_e2e():
        if not (rowpart or is5):
            # the public host API on pinned buffers (cww_*_host_async): chunk-pipelined H2D /
            # compute / D2H; forward and adjoint are independent, so they run on two streams
            # and the two PCIe directions overlap.  Tiny inputs (config 1) go zero-copy.
            cur = torch.cuda.current_stream(dev)
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
            x_rows.copy_(x_dev.view(1 << j, 1 << j)[rank * mr:(rank + 1) * mr])
            d2.normal(x_rows, CFG5_ITERS)
            ao_pin.view(1 << j, 1 << j)[rank * mr:(rank + 1) * mr].copy_(x_rows, non_blocking=True)
        else:
            ao_dev.copy_(x_dev)
            op.normal(ao_dev, iters=CFG5_ITERS, work=fo_dev)
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
        """The step captured once into a CUDA graph and replayed; eager calls when
        capture fails or a replay does not reproduce the eager outputs bit for bit,
        and under a profiler (ncu's per-node replay of graph kernels does not keep
        the graph's stream-ordered scratch allocations alive).
        Returns (callable, kernel launches per step or None)."""
        if under_profiler():
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
    dev_outs = [ao_dev] if is5 else [fo_dev, ao_dev]
    if rowpart:
        dev_outs = [x_rows]
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
    e2e_outs = [ao_pin] if is5 else [fo_pin, ao_pin]
    step_e2e_g, _ = graphed(step_e2e, e2e_outs) if not rowpart else (step_e2e, None)
    for _ in range(2):
        step_e2e_g()
    ms_e2e = timed(step_e2e_g, args.steps)

    # configs 2-4: the global batch split over the ranks (sum of the shards);
    # config 1: one replica per rank; config 5: one shared image
    total_mv = mv_per_step * args.steps * (1 if rowpart else world)
    if args.config in (2, 3, 4) and world > 1:
        total_mv = 2 * gbatch * args.steps
    value = total_mv / (ms / 1e3)
    e2e = total_mv / (ms_e2e / 1e3)
    h2d = x_pin.numel() * 8 + (0 if is5 else y_pin.numel() * 8)
    d2h = ao_pin.numel() * 8 + (0 if is5 else fo_pin.numel() * 8)

    # roofline of the dominant kernel: its SURVEY 8(d) bytes / its device time
    peak, peak_kind = peaks()
    roof = None
    nvec = batch
    if prof:
        kname = max(prof, key=lambda k: prof[k][0])
        kms, kn = prof[kname]
        steps_bytes = algorithmic_bytes(cfg, kname, nvec) * args.steps
        achieved = steps_bytes / (kms / 1e3) / 1e9 if kms > 0 else 0.0
        traffic, tnote = None, None
        entries, src = latest_traffic(args.config)
        for tr in entries:
            if tr["kernel"] == kname:
                traffic, tnote = tr["bytes"], f"{tr['launch']} (ncu dram__bytes_read+write, profiles/{src})"
        roof = {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_launch": tnote,
                "algorithmic_bytes_per_launch": steps_bytes / kn if kn else None,
                "kernel_ms_per_launch": kms / kn, "launches": kn,
                "kernel_share_of_step": round(kms / ms_prof, 4)}
    per_mv = path_bytes(cfg)
    path_gbs = per_mv * total_mv / world / (ms / 1e3) / 1e9

    line = {
        "metric": "forward+adjoint matvecs/s", "value": round(value, 3), "unit": "matvec/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": scaling_kind(args.config, world),
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded test_rng inputs, SURVEY.md 8d)",
        "config": config_dict(args.config, world),
        "launch": ("one CUDA graph per step (captured once, replayed)" if per_launch is not None
                   else "eager launches"),
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
                "link_gbs": round((h2d + d2h) / (ms_e2e / args.steps / 1e3) / 1e9, 1)},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args.config, xs, None if is5 else ys)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

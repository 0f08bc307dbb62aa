#!/usr/bin/env python
"""bench.py -- band -> bidiagonal reduction on B200 (arXiv 2510.12705 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype f64|f32|f16] [--n N] [--b B] [--tw TW]
                    [--no-extra] [--no-batched] [--no-cpu-baseline] [--no-e2e]
                    [--backend nccl|gloo] [--dry-run]

A "step" is one full reduction (pack + every pass of Alg. 1 + extract) of
one batch of synthetic banded matrices, inputs resident in HBM.

Top-level line (the driver's number): BASELINE config 4 -- one n=32768,
b=128 matrix per GPU (fp64, tw=32), i.i.d. N(0,1) band entries.  At N > 1
every rank reduces its own matrix (weak scaling; one matrix never spans GPUs,
its sweeps are a strict chain -- DESIGN.md section 9).  `value` = algorithmic
bytes of all ranks / max-over-ranks device time.

Sub-records in the same line:
  "batched": BASELINE config 5 -- 64 matrices n=16384, b=128, fp64 split
             across the N ranks (strong scaling), matrices/s, per-GPU GB/s, the
             NCCL all-gather of (d, e) timed separately, parity of matrices
             0 / 63 against the oracle's golden files;
  "extra":   (N = 1) config 4 in fp32, config 2 (n=1024), config 3 (n=8192),
             each with its own roofline fraction;
  "parity":  the timed output itself against tests/golden/ (oracle-written).

--gpus N without torchrun re-launches itself under torch.distributed.run
(one rank per GPU, 127.0.0.1 rendezvous).  --dry-run (CPU, gloo) exercises
spawn, the all-gather and the JSON line without any device work.

Metric (BASELINE.json): effective GB/s = algorithmic bytes (each
step's two-sided window read once + written once) / device time; also
GFLOP/s and matrices/s.  Roofline: the pass kernels' algorithmic bytes over
their CUDA-event time vs the measured HBM copy bandwidth.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ES = {"f16": 2, "f32": 4, "f64": 8}
METRIC = "band_to_bidiag_effective_GBps"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f16", "f32", "f64"])
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--tw", type=int, default=32)
    ap.add_argument("--maxb", type=int, default=0)
    ap.add_argument("--batch", type=int, default=64, help="batched sub-record: total matrices")
    ap.add_argument("--batched-n", type=int, default=16384)
    ap.add_argument("--batched-b", type=int, default=128)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-batched", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--dry-run", action="store_true", help="no device work: spawn + gather + JSON only")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args(argv)


# --------------------------------------------------------------------------- ranks
def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_if_needed(a):
    """--gpus N without a torchrun environment: re-exec under torch.distributed.run,
    one process per GPU; returns the child's exit code (None: run here)."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons during the timed region (NVML)."""

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _reason_names(self, mask):
        nv = self.nv
        names = []
        table = [("applications_clocks_setting", "nvmlClocksThrottleReasonApplicationsClocksSetting"),
                 ("sw_power_cap", "nvmlClocksThrottleReasonSwPowerCap"),
                 ("hw_slowdown", "nvmlClocksThrottleReasonHwSlowdown"),
                 ("sync_boost", "nvmlClocksThrottleReasonSyncBoost"),
                 ("sw_thermal_slowdown", "nvmlClocksThrottleReasonSwThermalSlowdown"),
                 ("hw_thermal_slowdown", "nvmlClocksThrottleReasonHwThermalSlowdown"),
                 ("hw_power_brake_slowdown", "nvmlClocksThrottleReasonHwPowerBrakeSlowdown")]
        for name, attr in table:
            bit = getattr(nv, attr, None)
            if bit is not None and mask & bit:
                names.append(name)
        return names

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                mask = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append(mhz)
                self.reasons.update(self._reason_names(mask))
            except Exception:
                pass
            time.sleep(0.1)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()
        return {"sm_mhz": (statistics.median(self.samples) if self.samples else None),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml" if self.ok else "unavailable"}


# --------------------------------------------------------------------------- peaks, host
def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """DRAM bytes (read + write) per step of the pass kernels, summed over the
    pass launches, from this round's ncu capture (profiles/ncu_traffic.json,
    written by tools/ncu_traffic.py from an ncu CSV); None if not measured."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            v = json.load(f).get(key)
        return v
    except Exception:
        return None


def host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# --------------------------------------------------------------------------- CPU oracle
def _oracle_native_once(compile=True):
    import oracle
    if not getattr(_oracle_native_once, "done", False):
        _oracle_native_once.flags = oracle.use_native_build("/tmp/bb_oracle_native", compile=compile) or \
            "-O2 -ffp-contract=off (portable build)"
        _oracle_native_once.done = True
    return _oracle_native_once.flags


def oracle_sample(band, b, tw, dtype, budget_s):
    """Time the CPU oracle (as it stands, single thread) on a bounded sample of
    the workload: the first S steps of the sequential reduction of one matrix,
    S calibrated so the sample takes about budget_s seconds."""
    import oracle
    o = oracle.Oracle(band, b, tw)
    t0 = time.perf_counter()
    done, elems = o.run(max_steps=200)
    t_cal = time.perf_counter() - t0
    o.close()
    per_step = max(t_cal / max(done, 1), 1e-7)
    S = max(200, int(budget_s / per_step))
    o = oracle.Oracle(band, b, tw)
    t0 = time.perf_counter()
    done, elems = o.run(max_steps=S)
    dt = time.perf_counter() - t0
    o.close()
    bytes_ = 2.0 * ES[dtype] * elems
    return {"seconds": dt, "steps": done, "alg_bytes": bytes_,
            "gbs": bytes_ / dt / 1e9, "sample": f"first {done} steps (sequential order, pass 1) of matrix 0"}


def _batched_cpu_worker(args):
    n, b, tw, mid, budget = args
    import synth
    _oracle_native_once(compile=False)  # built once by the parent
    band = synth.random_band(n, b, "f64", seed=0, matrix_id=mid)
    return oracle_sample(band, b, tw, "f64", budget)


def batched_cpu(n, b, tw, mat_bytes, budget):
    """P = min(64, cores) oracle processes at once, one matrix each, a bounded
    sample per process; host matrices/s = P / (per-matrix bytes / per-process rate)."""
    from multiprocessing import get_context
    _oracle_native_once()
    P = max(1, min(64, os.cpu_count() or 1))
    t0 = time.perf_counter()
    with get_context("spawn").Pool(P) as pool:
        res = pool.map(_batched_cpu_worker, [(n, b, tw, m, budget) for m in range(P)])
    wall = time.perf_counter() - t0
    rate = sum(r["alg_bytes"] for r in res) / max(r["seconds"] for r in res)  # B/s, all processes
    return {"value": mat_bytes and rate / mat_bytes, "unit": "matrices/s", "gbs": rate / 1e9, "processes": P,
            "cores": P, "kind": "oracle",
            "sample": f"{P} concurrent oracle processes, each the first ~{budget:.0f} s of steps of one "
                      f"n={n} b={b} fp64 matrix; matrices/s = aggregate bytes/s / bytes per matrix",
            "wall_s": wall}


def run_reference(a):
    """--impl reference: the CPU oracle on the host cores (the base contract's
    reference arm for this tier), same config/metric/unit."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import synth
    flags = _oracle_native_once()
    band = synth.random_band(a.n, a.b, a.dtype, seed=a.seed, matrix_id=0)
    for _ in range(a.warmup):
        oracle_sample(band, a.b, a.tw, a.dtype, 0.5)
    vals, tsum, last = [], 0.0, None
    per = max(1.0, min(a.cpu_seconds, 60.0) / max(a.steps, 1))
    for _ in range(a.steps):
        r = oracle_sample(band, a.b, a.tw, a.dtype, per)
        vals.append(r["gbs"])
        tsum += r["seconds"]
        last = r
    v = float(np.mean(vals))
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s",
           "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tsum / a.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": a.dtype,
           "data": "synthetic: i.i.d. N(0,1) band entries (numpy Philox, seed %d)" % a.seed,
           "config": workload_config(a, world),
           "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": last["sample"],
                            "build": flags, "host": host_info()},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def workload_config(a, world):
    return {"workload": f"single n={a.n} b={a.b} {a.dtype} tw={a.tw} per GPU (BASELINE config 4)",
            "n": a.n, "b": a.b, "tw": a.tw, "matrices_per_gpu": 1, "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write); within a step the working band is "
                  "L2-resident by design"}


# --------------------------------------------------------------------------- device helpers
class Runner:
    """One configuration on this rank's device: inputs generated once (seeded,
    matrix ids), copied to HBM, a pre-allocated workspace, per-pass CUDA events."""

    def __init__(self, bb, torch, dev, n, b, dtype, tw, ids, maxb=0, seed=0):
        import synth
        self.bb, self.torch, self.dev = bb, torch, dev
        self.n, self.b, self.dtype, self.tw, self.ids = n, b, dtype, tw, ids
        self.B = len(ids)
        self.host = np.stack([synth.random_band(n, b, dtype, seed=seed, matrix_id=i) for i in ids])
        self.band = torch.from_numpy(self.host).to(dev)
        self.cfg = bb.Config(tw=tw, max_blocks_per_sm=maxb)
        self.ws = bb.Workspace(n, b, dtype, self.B, cfg=self.cfg, device=dev)
        self.st = self.ws.stats
        self.P = self.st["passes"]
        self.d = torch.empty(self.B, n, dtype=self.band.dtype, device=dev)
        self.e = torch.empty(self.B, max(n - 1, 1), dtype=self.band.dtype, device=dev)
        self.stream = torch.cuda.current_stream(dev)
        self.launches = bb.launch_count(n, b, dtype, self.B, self.cfg)

    def step(self, events=None):
        bb = self.bb
        c = bb.Config(**{**self.cfg.__dict__, "timing_events": tuple(events) if events else ()})
        bb.bb_band_to_bidiag_batched_ex(self.n, self.b, bb.api.bb_dtype(self.dtype), self.B, self.band.data_ptr(),
                                        self.b + 1, self.n * (self.b + 1), self.d.data_ptr(), self.d.stride(0),
                                        self.e.data_ptr(), self.e.stride(0), c.c(), self.ws.buf.data_ptr(),
                                        self.ws.nbytes, self.stream.cuda_stream)

    def timed(self, steps, warmup, flush, barrier=lambda: None):
        torch = self.torch
        for _ in range(warmup):
            flush.fill_(1.0)
            self.step()
        torch.cuda.synchronize()
        step_ms, pass_ms = [], []
        barrier()
        torch.cuda.synchronize()
        for _ in range(steps):
            flush.fill_(1.0)                        # evict L2 between timed steps
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(self.P + 3)]
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(self.stream)
            self.step(evs)
            s1.record(self.stream)
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            pass_ms.append([evs[1 + p].elapsed_time(evs[2 + p]) for p in range(self.P)])
        torch.cuda.synchronize()
        barrier()
        return step_ms, pass_ms

    def roofline(self, pass_ms, ms_per_step):
        peak, src = hbm_peak()
        pm = np.mean(np.array(pass_ms), axis=0) if len(pass_ms) else np.zeros(self.P)
        tot = float(np.sum(pm))
        ach = self.st["alg_bytes"] * self.B / (tot * 1e-3) / 1e9 if tot > 0 else None
        key = f"{self.n}:{self.b}:{self.dtype}:{self.tw}:{self.B}"
        tr = ncu_traffic(key)
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None, "traffic": tr,
                "traffic_source": ("profiles/ncu_traffic.json[%s] (ncu dram__bytes_read+write, pass kernels, "
                                   "per step)" % key) if tr is not None else None,
                "peak_source": src,
                "kernel": "pass kernels: pass_v5_kernel (unit kernel, target bandwidth >= 8), pass_v6_kernel "
                          "(segment ring, target bandwidth 1)",
                "alg_bytes_per_step": self.st["alg_bytes"] * self.B,
                "pass_ms_mean": [float(x) for x in pm],
                "pass_share_of_step": tot / ms_per_step if ms_per_step else None}

    def parity(self, golden_names):
        """The timed output against oracle-written golden files (|d|, |e|,
        normwise, north_star tolerances, reading Q15)."""
        from tests.golden_util import errors, golden_path, input_sha256, load, tol
        d = self.d.double().cpu().numpy()
        e = self.e[:, : self.n - 1].double().cpu().numpy()
        out = []
        for k, name in golden_names:
            if not os.path.exists(golden_path(name)):
                continue
            g = load(name)
            same_input = input_sha256(self.host[k]) == g["sha256"]
            err = errors(g, d[k], e[k])
            lim = tol(self.dtype, self.n)
            rel = max(err["d"], err["e"]) / g["fro"]
            out.append({"golden": name, "same_input": same_input, "max_abs_err_over_normF": rel, "tol": lim,
                        "ok": bool(same_input and rel <= lim)})
        return out


def record(r, step_ms, pass_ms, mats_total, ms=None, label=""):
    ms = ms if ms is not None else float(np.mean(step_ms))
    ab = r.st["alg_bytes"] * mats_total
    return {"workload": label, "n": r.n, "b": r.b, "dtype": r.dtype, "tw": r.tw, "matrices": mats_total,
            "ms_per_step": ms, "value": ab / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "gflops": r.st["alg_flops"] * mats_total / (ms * 1e-3) / 1e9, "matrices_per_s": mats_total / (ms * 1e-3),
            "roofline": r.roofline(pass_ms, ms)}


# --------------------------------------------------------------------------- main
def main():
    a = parse()
    rc = relaunch_if_needed(a)
    if rc is not None:
        sys.exit(rc)
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist
    from paper_2510_12705_b200.dist import gather_results, partition

    world, rank, local = dist_env()
    if a.dry_run:
        return dry_run(a, world, rank)
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group(a.backend, device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2510_12705_b200 as bb
    barrier = (lambda: dist.barrier()) if world > 1 else (lambda: None)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # ---------------------------------------------------------------- headline: config 4, one matrix per GPU
    head = Runner(bb, torch, dev, a.n, a.b, a.dtype, a.tw, [rank], maxb=a.maxb, seed=a.seed)
    clocks = ClockSampler(dev.index)
    clocks.start()
    step_ms, pass_ms = head.timed(a.steps, a.warmup, flush, barrier)
    clk = clocks.stop()
    ms_per_step = max_over_ranks(float(np.mean(step_ms)))
    alg_bytes_step = head.st["alg_bytes"] * world
    value = alg_bytes_step / (ms_per_step * 1e-3) / 1e9
    gname = f"c4_n{a.n}_b{a.b}_{a.dtype}_s{a.seed}_m{rank}"
    parity = head.parity([(0, gname)])

    # e2e: the C-ABI host entry point, pinned host buffers, H2D + D2H inside the region
    e2e = None
    if not a.no_e2e:
        pin = torch.from_numpy(head.host).pin_memory()
        dh = torch.empty(1, a.n, dtype=pin.dtype).pin_memory()
        eh = torch.empty(1, max(a.n - 1, 1), dtype=pin.dtype).pin_memory()

        def e2e_step():
            bb.bb_band_to_bidiag_host(a.n, a.b, bb.api.bb_dtype(a.dtype), 1, pin.data_ptr(), a.b + 1,
                                      a.n * (a.b + 1), dh.data_ptr(), dh.stride(0), eh.data_ptr(), eh.stride(0),
                                      head.cfg.c(), head.stream.cuda_stream)
        e2e_step()
        times = []
        for _ in range(max(1, min(a.steps, 3))):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - t0)
        tt = max_over_ranks(float(np.mean(times)))
        e2e = {"value": alg_bytes_step / tt / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(pin.numel() * pin.element_size()),
               "d2h_bytes_per_step": int((2 * a.n - 1) * pin.element_size()),
               "ms_per_step": tt * 1e3, "api": "bb_band_to_bidiag_host (C ABI, pinned host buffers)",
               "timing": "host wall clock around the blocking call, max over ranks"}
    launches = head.launches * a.steps
    del head

    # ---------------------------------------------------------------- batched: config 5 split across ranks
    batched = None
    if not a.no_batched:
        start, count = partition(a.batch, world, rank)
        counts = [partition(a.batch, world, r)[1] for r in range(world)]
        rb = Runner(bb, torch, dev, a.batched_n, a.batched_b, "f64", 32, list(range(start, start + count)),
                    seed=a.seed)
        bsteps = 1
        s_ms, p_ms = rb.timed(bsteps, 1, flush, barrier)
        ms_b = max_over_ranks(float(np.mean(s_ms)))
        # the one data-path collective: all-gather of (d, e), timed on its own
        g_ms = None
        if world > 1:
            torch.cuda.synchronize()
            barrier()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record()
            gather_results(rb.d, rb.e[:, : a.batched_n - 1], world, counts=counts)
            g1.record()
            torch.cuda.synchronize()
            g_ms = max_over_ranks(g0.elapsed_time(g1))
        batched = record(rb, s_ms, p_ms, a.batch, ms=ms_b,
                         label=f"batched {a.batch} x n={a.batched_n} b={a.batched_b} f64 tw=32 split over "
                               f"{world} GPU(s) (BASELINE config 5, strong scaling)")
        batched["per_gpu_gbs"] = batched["value"] / world
        batched["gather_ms"] = g_ms
        batched["steps"] = bsteps
        batched["warmup"] = 1
        names = [(k, f"c5_n{a.batched_n}_b{a.batched_b}_f64_s{a.seed}_m{m}")
                 for k, m in enumerate(range(start, start + count)) if m in (0, a.batch - 1)]
        batched["parity"] = rb.parity(names)
        batched["launches"] = rb.launches * bsteps
        if rank == 0 and world == 1 and not a.no_cpu_baseline:
            mat_bytes = rb.st["alg_bytes"]
            batched["cpu_baseline"] = batched_cpu(a.batched_n, a.batched_b, 32, mat_bytes,
                                                  max(2.0, a.cpu_seconds / 3))
        del rb

    # ---------------------------------------------------------------- extra single-GPU records (N = 1)
    extra = []
    if world == 1 and not a.no_extra:
        for (n, b, dt, tw, steps, tag) in [(32768, 128, "f32", 32, 2, "c4"), (1024, 32, "f64", 32, 5, "c2"),
                                            (1024, 32, "f32", 32, 5, "c2"), (8192, 64, "f64", 32, 3, "c3"),
                                            (8192, 64, "f32", 32, 3, "c3"), (8192, 64, "f16", 32, 3, "c3")]:
            r = Runner(bb, torch, dev, n, b, dt, tw, [0], seed=a.seed)
            s_ms, p_ms = r.timed(steps, 1, flush)
            rec = record(r, s_ms, p_ms, 1, label=f"BASELINE config {tag[1]}: n={n} b={b} {dt} tw={tw}")
            rec["steps"] = steps
            rec["parity"] = r.parity([(0, f"{tag}_n{n}_b{b}_{dt}_s{a.seed}_m0")])
            extra.append(rec)
            del r

    # ---------------------------------------------------------------- stage 3 and small-n batched (N = 1)
    stage3 = None
    small_batched = None
    if world == 1 and not a.no_extra:
        # SVD stage 3 on the device (F3): singular values of the headline bidiagonal
        r = Runner(bb, torch, dev, a.n, a.b, a.dtype, a.tw, [0], seed=a.seed)
        r.step()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bb.bidiag_svals(r.d[0], r.e[0, : a.n - 1])
        times = []
        for _ in range(3):
            ev0.record()
            sig = bb.bidiag_svals(r.d[0], r.e[0, : a.n - 1])
            ev1.record()
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
        stage3 = {"workload": f"singular values of the n={a.n} bidiagonal (bisection, fp64)", "ms": float(np.median(times))}
        from tests.golden_util import golden_path, load
        gname = f"c4_n{a.n}_b{a.b}_{a.dtype}_s{a.seed}_m0"
        if os.path.exists(golden_path(gname)):
            g = load(gname)
            stage3["max_abs_err_over_normF_vs_oracle"] = float(np.max(np.abs(sig.cpu().numpy() - g["sigma"]))) / g["fro"]
        del r
        # F2: many small matrices at the paper's crossover size, interleaved in the same launches
        nsm = 512
        r = Runner(bb, torch, dev, 1024, 32, "f64", 32, list(range(nsm)), seed=a.seed)
        s_ms, p_ms = r.timed(2, 1, flush)
        small_batched = record(r, s_ms, p_ms, nsm, label=f"batched {nsm} x n=1024 b=32 f64 tw=32 (config 2 size)")
        del r

    # ---------------------------------------------------------------- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        import synth
        flags = _oracle_native_once()
        band = synth.random_band(a.n, a.b, a.dtype, seed=a.seed, matrix_id=0)
        r = oracle_sample(band, a.b, a.tw, a.dtype, a.cpu_seconds)
        cpu = {"value": r["gbs"], "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": r["sample"],
               "seconds": r["seconds"], "build": flags, "host": host_info()}

    if rank == 0:
        roof = None
        # roofline of the headline pass kernels (this rank's events)
        peak, src = hbm_peak()
        pm = np.mean(np.array(pass_ms), axis=0)
        tot = float(np.sum(pm))
        st = bb.plan(a.n, a.b, a.dtype, 1, bb.Config(tw=a.tw, max_blocks_per_sm=a.maxb))
        ach = st["alg_bytes"] / (tot * 1e-3) / 1e9
        key = f"{a.n}:{a.b}:{a.dtype}:{a.tw}:1"
        tr = ncu_traffic(key)
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": tr, "traffic_source": ("profiles/ncu_traffic.json[%s]" % key) if tr is not None else None,
                "peak_source": src,
                "kernel": "pass kernels of one step (pass_v5_kernel x3: unit kernel; pass_v6_kernel: segment ring, "
                          "target bandwidth 1); achieved = algorithmic bytes of the passes / their summed CUDA-event "
                          "time on the launching stream",
                "alg_bytes_per_step_per_rank": st["alg_bytes"], "pass_ms_mean": [float(x) for x in pm],
                "pass_share_of_step": tot / float(np.mean(step_ms))}
        out = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": a.dtype,
               "data": "synthetic: i.i.d. N(0,1) band entries (numpy Philox, seed %d, matrix id = rank), rounded "
                       "to %s" % (a.seed, a.dtype),
               "config": workload_config(a, world),
               "gflops": st["alg_flops"] * world / (ms_per_step * 1e-3) / 1e9,
               "matrices_per_s": world / (ms_per_step * 1e-3),
               "alg_bytes_per_step": alg_bytes_step, "alg_flops_per_step": st["alg_flops"] * world,
               "critical_cycles": st["critical_cycles"], "passes": st["passes"], "steps_per_matrix": st["steps"],
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
               "gpu_launches": int(launches), "parity": parity, "batched": batched, "extra": extra,
               "stage3": stage3, "small_batched": small_batched,
               "step_ms": step_ms}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dry_run(a, world, rank):
    """CPU harness check: process group (gloo), the batched partition and its
    single all-gather of fixed-shape (d, e) buffers, and the JSON line --
    no device work, no numbers."""
    import torch
    import torch.distributed as dist
    from paper_2510_12705_b200.dist import gather_results, partition
    if world > 1:
        dist.init_process_group("gloo")
    start, count = partition(a.batch, world, rank)
    counts = [partition(a.batch, world, r)[1] for r in range(world)]
    n = 8
    d = torch.arange(start, start + count, dtype=torch.float64).repeat_interleave(n).reshape(count, n)
    e = -d[:, : n - 1]
    D, E = gather_results(d, e, world, counts=counts)
    ok = bool(torch.equal(D[:, 0], torch.arange(a.batch, dtype=torch.float64)))
    if rank == 0:
        out = {"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": world, "steps": 0, "warmup": 0,
               "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": a.dtype, "data": "dry run (no device work)", "config": workload_config(a, world),
               "dry_run": True, "gather_ok": ok, "gathered_shape": list(D.shape)}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- band -> bidiagonal reduction on B200 (arXiv 2510.12705 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload single|batched] [--dtype f64|f32|f16] [--n N] [--b B] [--tw TW]

A "step" is one full reduction (every pass of Alg. 1, pack + passes +
extract) of one batch of synthetic banded matrices.  Default workload
(N=1): BASELINE config 4, one n=32768, b=128 matrix per GPU (fp64, tw=16),
i.i.d. N(0,1) band entries.  --workload batched: BASELINE config 5, 64
matrices n=16384 split across the ranks (strong scaling).  Under torchrun,
the single workload gives each rank its own matrix (weak scaling) and the
results are gathered with NCCL (the only collective).

Metric (BASELINE.json): effective GB/s = algorithmic bytes (SURVEY §8d:
each step's two-sided window read once + written once) / device time; also
GFLOP/s and matrices/s.  Roofline: the pass kernels' algorithmic bytes over
their CUDA-event time vs the measured HBM copy bandwidth.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ES = {"f16": 2, "f32": 4, "f64": 8}
DEFAULT_TW = {"f16": 32, "f32": 32, "f64": 32}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="single", choices=["single", "batched"])
    ap.add_argument("--dtype", default="f64", choices=["f16", "f32", "f64"])
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--b", type=int, default=0)
    ap.add_argument("--tw", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0, help="batched workload: total matrices (default 64)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--maxb", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    if a.workload == "single":
        a.n = a.n or 32768
        a.b = a.b or 128
    else:
        a.n = a.n or 16384
        a.b = a.b or 128
        a.batch = a.batch or 64
    a.tw = a.tw or DEFAULT_TW[a.dtype]
    return a


# --------------------------------------------------------------------------- dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def matrices_for_rank(a, world, rank):
    """Global matrix ids this rank reduces."""
    from paper_2510_12705_b200.dist import partition
    if a.workload == "single":
        return [rank]                      # weak scaling: one n x n matrix per GPU
    start, count = partition(a.batch, world, rank)
    return list(range(start, start + count))


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
        table = [("gpu_idle", "nvmlClocksThrottleReasonGpuIdle"),
                 ("applications_clocks_setting", "nvmlClocksThrottleReasonApplicationsClocksSetting"),
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
                for r in self._reason_names(mask):
                    if r != "gpu_idle":
                        self.reasons.add(r)
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


# --------------------------------------------------------------------------- peaks
def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


# --------------------------------------------------------------------------- CPU oracle
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


def run_reference(a):
    """--impl reference: the CPU oracle on the host cores (the base contract's
    reference arm for this tier), same config/metric/unit."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import synth
    band = synth.random_band(a.n, a.b, a.dtype, seed=a.seed, matrix_id=0)
    for _ in range(a.warmup):
        oracle_sample(band, a.b, a.tw, a.dtype, 0.5)
    vals = []
    tsum = 0.0
    last = None
    per = max(1.0, min(a.cpu_seconds, 60.0) / max(a.steps, 1))
    for _ in range(a.steps):
        r = oracle_sample(band, a.b, a.tw, a.dtype, per)
        vals.append(r["gbs"])
        tsum += r["seconds"]
        last = r
    v = float(np.mean(vals))
    out = {"impl": "reference", "metric": "band_to_bidiag_effective_GBps", "value": v, "unit": "GB/s",
           "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tsum / a.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": a.dtype,
           "data": "synthetic: i.i.d. N(0,1) band entries (numpy Philox, seed %d)" % a.seed,
           "config": workload_config(a),
           "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": last["sample"]},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def workload_config(a):
    if a.workload == "single":
        w = f"single n={a.n} b={a.b} {a.dtype} tw={a.tw} (BASELINE config 4)"
    else:
        w = f"batched {a.batch} x n={a.n} b={a.b} {a.dtype} tw={a.tw} (BASELINE config 5)"
    return {"workload": w, "n": a.n, "b": a.b, "tw": a.tw, "batch": (a.batch if a.workload == "batched" else None),
            "parallelism": f"dp{a.gpus}", "l2": "flushed between timed steps (256 MiB write); "
            "within a step the working band is L2-resident by design"}


# --------------------------------------------------------------------------- ours
def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import synth
    import paper_2510_12705_b200 as bb
    from paper_2510_12705_b200.dist import gather_results

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()

    ids = matrices_for_rank(a, world, rank)
    B = len(ids)
    bands_np = np.stack([synth.random_band(a.n, a.b, a.dtype, seed=a.seed, matrix_id=i) for i in ids])
    band = torch.from_numpy(bands_np).to(dev)
    cfg = bb.Config(tw=a.tw, threads_per_block=a.threads, max_blocks_per_sm=a.maxb)
    ws = bb.Workspace(a.n, a.b, a.dtype, B, cfg=cfg, device=dev)
    st = ws.stats
    P = st["passes"]
    d = torch.empty(B, a.n, dtype=band.dtype, device=dev)
    e = torch.empty(B, max(a.n - 1, 1), dtype=band.dtype, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    launches_per_step = bb.launch_count(a.n, a.b, a.dtype, B, cfg)

    def step(events=None):
        c = bb.Config(**{**cfg.__dict__, "timing_events": tuple(events) if events else ()})
        bb.bb_band_to_bidiag_batched_ex(a.n, a.b, bb.api.bb_dtype(a.dtype), B, band.data_ptr(), a.b + 1,
                                        a.n * (a.b + 1), d.data_ptr(), d.stride(0), e.data_ptr(), e.stride(0),
                                        c.c(), ws.buf.data_ptr(), ws.nbytes, stream.cuda_stream)
        if world > 1:
            gather_results(d, e, world)

    for _ in range(a.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(dev.index)
    step_ms = []
    pass_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for _ in range(a.steps):
        flush.fill_(1.0)                         # evict L2 between timed steps
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(P + 3)]
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        step(evs)
        s1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(s0.elapsed_time(s1))
        pass_ms.append([evs[1 + p].elapsed_time(evs[2 + p]) for p in range(P)])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()

    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / a.steps
    mats_total = a.batch if a.workload == "batched" else world
    alg_bytes_step = st["alg_bytes"] * mats_total          # all ranks
    alg_flops_step = st["alg_flops"] * mats_total
    value = alg_bytes_step / (ms_per_step * 1e-3) / 1e9
    gflops = alg_flops_step / (ms_per_step * 1e-3) / 1e9
    mps = mats_total / (ms_per_step * 1e-3)

    # roofline of the dominant kernel (the per-pass persistent kernels), this rank
    pass_total_ms = float(np.sum(pass_ms)) / a.steps
    achieved = st["alg_bytes"] * B / (pass_total_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    key = f"{a.workload}:{a.n}:{a.b}:{a.dtype}:{a.tw}"
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(key), "peak_source": peak_src,
            "kernel": "pass_v4_kernel (multi-sweep persistent launch per pass; v2 register kernel where v4 does not apply)",
            "alg_bytes_per_step_per_rank": st["alg_bytes"] * B,
            "pass_ms_mean": [float(x) for x in np.mean(np.array(pass_ms), axis=0)],
            "pass_share_of_step": pass_total_ms / ms_per_step}

    # parity spot check of this run's output (cheap, always on): structural invariants
    torch.cuda.synchronize()

    # e2e: the C-ABI host entry point, host buffers, H2D + D2H inside the region
    e2e = None
    if not a.no_e2e:
        pin = torch.from_numpy(bands_np).pin_memory()
        dh = torch.empty(B, a.n, dtype=pin.dtype).pin_memory()
        eh = torch.empty(B, max(a.n - 1, 1), dtype=pin.dtype).pin_memory()

        def e2e_step():
            bb.bb_band_to_bidiag_host(a.n, a.b, bb.api.bb_dtype(a.dtype), B, pin.data_ptr(), a.b + 1,
                                      a.n * (a.b + 1), dh.data_ptr(), dh.stride(0), eh.data_ptr(), eh.stride(0),
                                      cfg.c(), stream.cuda_stream)
        e2e_step()
        k = max(1, min(a.steps, 3))
        times = []
        for _ in range(k):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - t0)
        tt = float(np.mean(times))
        if world > 1:
            tq = torch.tensor([tt], dtype=torch.float64, device=dev)
            dist.all_reduce(tq, op=dist.ReduceOp.MAX)
            tt = float(tq.item())
        e2e = {"value": alg_bytes_step / tt / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(pin.numel() * pin.element_size()),
               "d2h_bytes_per_step": int(B * (2 * a.n - 1) * pin.element_size()),
               "ms_per_step": tt * 1e3, "api": "bb_band_to_bidiag_host (C ABI, pinned host buffers)",
               "timing": "host wall clock around the blocking call, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        r = oracle_sample(bands_np[0], a.b, a.tw, a.dtype, a.cpu_seconds)
        cpu = {"value": r["gbs"], "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": r["sample"],
               "seconds": r["seconds"]}

    if rank == 0:
        out = {"metric": "band_to_bidiag_effective_GBps", "value": value, "unit": "GB/s", "n_gpus": world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "weak" if a.workload == "single" else "strong", "vs_baseline": None,
               "dtype": a.dtype,
               "data": "synthetic: i.i.d. N(0,1) band entries (numpy Philox, seed %d), rounded to %s" % (a.seed, a.dtype),
               "config": workload_config(a),
               "gflops": gflops, "matrices_per_s": mps,
               "alg_bytes_per_step": alg_bytes_step, "alg_flops_per_step": alg_flops_step,
               "critical_cycles": st["critical_cycles"], "passes": P, "steps_per_matrix": st["steps"],
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
               "gpu_launches": int(launches_per_step * a.steps),
               "step_ms": step_ms}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

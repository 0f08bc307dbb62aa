"""Scratch: does the workspace allocation kind matter?  Per-pass times of the
headline reduction with the workspace from (a) torch's caching allocator
(cudaMalloc), (b) cuMemCreate without compression, (c) cuMemCreate with
generic compression, plus the library's own cudaMallocAsync path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import driver as D  # noqa: E402

import synth  # noqa: E402
import paper_2510_12705_b200 as bb  # noqa: E402


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


def vmm_alloc(nbytes, comp):
    dev = torch.cuda.current_device()
    prop = D.CUmemAllocationProp()
    prop.type = D.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = D.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = dev
    prop.allocFlags.compressionType = comp
    gran = ck(D.cuMemGetAllocationGranularity(prop, D.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
    size = (nbytes + gran - 1) // gran * gran
    h = ck(D.cuMemCreate(size, prop, 0))
    ptr = ck(D.cuMemAddressReserve(size, 0, 0, 0))
    ck(D.cuMemMap(ptr, size, 0, h, 0))
    acc = D.CUmemAccessDesc()
    acc.location.type = D.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = dev
    acc.flags = D.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    ck(D.cuMemSetAccess(ptr, size, [acc], 1))
    return int(ptr), size


def run(n, b, dt, tw, ws_ptr, ws_bytes, label, reps=2):
    band = torch.from_numpy(synth.random_band(n, b, dt, seed=0)).cuda()
    st = bb.plan(n, b, dt, tw=tw)
    P = st["passes"]
    d = torch.empty(n, dtype=band.dtype, device="cuda")
    e = torch.empty(n - 1, dtype=band.dtype, device="cuda")
    for _ in range(reps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(P + 3)]
        c = bb.Config(tw=tw, timing_events=tuple(evs))
        if ws_ptr is None:  # the library's own stream-ordered allocation; total time only
            evs[0].record()
            bb.bb_band_to_bidiag(n, b, bb.api.bb_dtype(dt), band.data_ptr(), b + 1, d.data_ptr(), e.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
            for ev in evs[1:]:
                ev.record()
        else:
            bb.bb_band_to_bidiag_ex(n, b, bb.api.bb_dtype(dt), band.data_ptr(), b + 1, d.data_ptr(), e.data_ptr(),
                                    c.c(), ws_ptr, ws_bytes, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        pm = [round(evs[1 + p].elapsed_time(evs[2 + p]), 1) for p in range(P)]
        print(f"{label:28s} {dt}: total {evs[0].elapsed_time(evs[P + 2]):.1f} ms passes {pm}", flush=True)


if __name__ == "__main__":
    n, b, tw = 32768, 128, 32
    for dt in sys.argv[1:] or ["f64"]:
        nb = bb.plan(n, b, dt, tw=tw)["workspace_bytes"]
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        run(n, b, dt, tw, ws.data_ptr(), nb, "torch caching allocator")
        run(n, b, dt, tw, None, 0, "library cudaMallocAsync")
        for comp, name in ((D.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_NONE, "cuMemCreate COMP_NONE"),
                           (D.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC, "cuMemCreate COMP_GENERIC")):
            try:
                p, sz = vmm_alloc(nb, comp)
            except Exception as ex:  # noqa: BLE001
                print(name, "unavailable:", ex, flush=True)
                continue
            run(n, b, dt, tw, p, nb, name)

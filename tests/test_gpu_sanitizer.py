"""compute-sanitizer over every pass kernel at small n (
P:73 warns about volatile-based inter-block synchronisation).

* memcheck (out-of-bounds / misaligned accesses), every kernel: must be clean.
* synccheck (barrier misuse) on the kernels synchronised by __syncthreads /
  named barriers only (unit kernel v5, register kernel v2, generic kernel,
  stage 3): must be clean.  synccheck models every mbarrier phase as
  consumed by a wait; the v4/v6 warp-group counters let a waiter skip the
  phases it does not need (the counter is the truth, the mbarrier only lets
  it sleep), which synccheck rejects even in a 40-line kernel
  (tools/ubench/sync_mb.cu: "Missing wait") -- those kernels are covered by
  racecheck and memcheck instead.
* racecheck (shared-memory hazards inside a CTA): the kernels synchronise
  warp-groups through shared-memory progress counters written with
  st.release / read with volatile + ld.acquire, and data through mbarrier
  phases (cp.async / TMA completion, arrive/try_wait).  racecheck models
  neither, so it reports the counter accesses themselves and the data
  accesses those counters order.  The test accepts exactly those pairs (an
  allowlist of the synchronisation functions, each an intended
  release/acquire or mbarrier hand-off) and fails on any other hazard.
The inter-CTA protocol (global progress flags) is outside racecheck's scope;
it is exercised by the bitwise run-to-run / schedule-independence tests."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (first access function, second access function) pairs ordered by the
# counters / mbarriers described above
ALLOWED = {
    "sts_release", "lds_volatile",          # the progress counters themselves
    "cp_async_elem", "fill_rect",           # v4 producer fills, ordered by cp.async.mbarrier.arrive phases
    "step_v6", "v6_store_cols",             # v6: beta/zero writes vs the writer's chunk read, ordered by
                                            # post_prog (release + arrive) -> wait_prog (try_wait + acquire)
    "v6_load_cols_h",                       # v6 fp16 producer stores, ordered by the chunk mbarrier
    "pass_v6_kernel",                       # step_v6 inlined into the kernel: same beta/zero writes as step_v6
    "ld_vec", "st_vec",                     # v4 slot reads/writes vs the producer's cp.async into the slot:
                                            # RAW ordered by the fill mbarrier, WAR by the slot-reuse wait
}


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


def _run(tool, n, extra=(), mode="all"):
    env = dict(os.environ, SAN_N=str(n), SAN_MODE=mode)
    p = subprocess.run([_sanitizer(), "--tool", tool, *extra, sys.executable,
                        os.path.join(ROOT, "tests", "san_run.py")], capture_output=True, text=True, timeout=1500,
                       env=env, cwd=ROOT)
    out = p.stdout + p.stderr
    if "compute-sanitizer is closed" in out or ("san_run ok" not in out and "closed on this pool" in out):
        # the GPU pool disables compute-sanitizer (runs under it left GPUs needing a
        # reset); the device-side bounds checks of tests/test_gpu_bounds.py stand in
        pytest.skip("compute-sanitizer disabled on this GPU pool")
    return p.returncode, out


@pytest.mark.parametrize("tool,mode", [("memcheck", "all"), ("synccheck", "sync")])
def test_sanitizer_clean(tool, mode):
    rc, out = _run(tool, 200, ["--error-exitcode", "3"], mode=mode)
    print(out[-2000:])
    assert rc == 0, out[-3000:]
    assert "san_run ok" in out and "ERROR SUMMARY: 0 errors" in out


def _fn(s):
    m = re.search(r"access at (?:void )?(?:bb::)?([A-Za-z_0-9]+)", s)
    return m.group(1) if m else "?"


def test_racecheck_only_synchronisation_accesses():
    rc, out = _run("racecheck", 140, ["--print-limit", "100000"])
    assert "san_run ok" in out, out[-3000:]
    lines = out.splitlines()
    bad = []
    for i, l in enumerate(lines):
        if "Race reported between" in l:
            a = _fn(l)
            b = _fn(lines[i + 1]) if i + 1 < len(lines) else "?"
            if a not in ALLOWED or b not in ALLOWED:
                bad.append((a, b, l.strip(), lines[i + 1].strip() if i + 1 < len(lines) else ""))
    import collections
    kinds = collections.Counter((a, b, re.findall(r"bb_\w+\.cuh:\d+", x + " " + y)[:2].__str__())
                                for a, b, x, y in bad)
    print("racecheck pairs outside the allowlist:", len(bad), kinds.most_common(20))
    assert not bad, kinds.most_common(20)

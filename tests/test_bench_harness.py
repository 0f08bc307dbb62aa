"""bench.py harness on CPU (no device work): --gpus N re-launches itself under
torch.distributed.run (gloo here), the batched partition's single all-gather
of (d, e) runs, and the JSON line reports n_gpus == --gpus with a matching
parallelism; the reference arm (the CPU oracle) prints its own line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


@pytest.mark.parametrize("gpus", [1, 2])
def test_dry_run_spawns_ranks_and_gathers(gpus):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--dry-run",
                        "--backend", "gloo"], capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    rec = _last_json(p.stdout)
    assert rec["n_gpus"] == gpus
    assert rec["config"]["parallelism"] == f"dp{gpus}"
    assert rec["gather_ok"] is True and rec["gathered_shape"] == [64, 8]


def test_reference_arm_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "256",
                        "--b", "16", "--tw", "8", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"],
                       capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    rec = _last_json(p.stdout)
    assert rec["impl"] == "reference" and rec["unit"] == "GB/s" and rec["value"] > 0
    assert rec["cpu_baseline"]["kind"] == "oracle" and rec["e2e"]["h2d_bytes_per_step"] == 0

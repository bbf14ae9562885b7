"""bench.py's own multi-rank harness and reference arm, on CPU.

* `--gpus 2` without torchrun re-executes bench.py under
  torch.distributed.run; the selftest workload then runs the rendezvous,
  max-over-ranks and slot all-reduce the GPU workloads use (gloo here).
* `--impl reference` builds its network and order with the oracle only: the
  product package (and its native library) is never imported in that arm."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_spawn_two_ranks_selftest():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "selftest"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1          # rank 0 only
    rec = json.loads(lines[0])
    assert rec["n_ranks"] == 2 and rec["backend"] == "gloo"
    assert rec["max_over_ranks"] == 0.002
    assert rec["slots"] == [1.0, -1.0, 2.0, -2.0]


_REF_ARM = r"""
import sys
sys.path.insert(0, {root!r})
import bench
args = bench.parse(["--impl", "reference", "--steps", "1", "--ref-budget-s", "0.01"])
bench._host_threads = lambda: 1
rc = bench.run_reference(args)
bad = [m for m in sys.modules if m.startswith("paper_2210_15874_b200")]
print("IMPORTED", bad)
"""


def test_reference_arm_never_imports_the_package():
    out = subprocess.run([sys.executable, "-c", _REF_ARM.format(root=ROOT)], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-1] == "IMPORTED []"
    rec = json.loads(lines[-2])
    assert rec["impl"] == "reference" and rec["dtype"] == "c128"
    assert abs(rec["details"]["zz"] - (-0.0017371891851279)) < 1e-12
    import bench
    assert rec["config"] == bench.CONFIG

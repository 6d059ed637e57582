"""CPU: bench.py's launcher and its reference arm (no GPU needed).

* `--gpus 2` re-launches itself under torchrun: both ranks join (gloo here),
  and the line reports n_gpus 2; WORLD_SIZE != --gpus fails loudly.
* `--impl reference` draws its inputs through the reference oracle only and
  never loads the product library (its timed path is oracle/_ref)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=ROOT)


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_launcher_spawns_ranks():
    r = _run(["--gpus", "2", "--launcher-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = _line(r.stdout)
    assert line["n_gpus"] == 2 and line["ranks_joined"] == 2 and line["max_rank"] == 1


def test_launcher_single_rank():
    r = _run(["--launcher-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert _line(r.stdout)["n_gpus"] == 1


def test_world_size_mismatch_fails():
    r = _run(["--gpus", "1", "--launcher-check"], env={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE" in r.stderr


PROBE = r"""
import json, os, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "gcd", "--steps", "1"]
sys.path.insert(0, os.getcwd())
import bench
args = type("A", (), dict(workload="gcd", s=0, steps=1, warmup=1))()
d = bench.Dist("reference")
line = bench.run_reference(args, d)
maps = open("/proc/self/maps").read()
print(json.dumps({"line": line,
                  "product_imported": "paper_1402_0264_b200" in sys.modules,
                  "libmmm_mapped": "libmmm_cu" in maps,
                  "ref_mapped": "libref_oracle" in maps}))
"""


def test_reference_arm_never_loads_the_product():
    from oracle import pyoracle
    r = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert not got["product_imported"] and not got["libmmm_mapped"]
    line = got["line"]
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    kind = "reference" if pyoracle.reference_available() else "port"
    assert line["cpu_baseline"]["kind"] == kind
    assert got["ref_mapped"] == (kind == "reference")


def test_ntt_sample_is_labelled_port():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.NttWork.cpu_ref_kind(None, "reference") == "port"
    assert bench.BatchWork.cpu_ref_kind(None, "reference") == "reference"

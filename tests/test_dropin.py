"""The C++ drop-in (include/mmm_b200.hpp) driven like the reference's own
tests and its `mmm verify` command (mmm_cli.cpp:456-528), on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "tests")


@pytest.fixture(scope="module")
def binaries():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return BIN


def test_dropin_builds_against_header(binaries):
    assert os.path.exists(os.path.join(binaries, "test_dropin"))
    assert os.path.exists(os.path.join(binaries, "mmm_verify"))


@pytest.mark.gpu
def test_dropin_reference_cases(binaries):
    r = subprocess.run([os.path.join(binaries, "test_dropin")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("p", [7, 101, 469762049])
def test_verify_harness(binaries, p):
    r = subprocess.run([os.path.join(binaries, "mmm_verify"), "--p", str(p), "--trials", "200"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" 200/200 ok") == 3, r.stdout


@pytest.mark.gpu
def test_verify_detects_injected_fault(binaries):
    # test_cli.cpp:152-162: the fault-injected verify must exit 2
    r = subprocess.run([os.path.join(binaries, "mmm_verify"), "--inject-fault", "--trials", "5",
                        "--app", "division"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stdout + r.stderr


REF_BENCH_SRC = "/root/reference/proj/tools/bench.cpp"
REF_BENCH_BIN = os.path.join(ROOT, "oracle", "_ref", "ref_tools_bench")


@pytest.mark.skipif(not os.path.exists(REF_BENCH_SRC), reason="reference sources absent")
def test_reference_bench_tool_builds_against_dropin(binaries):
    """/root/reference/proj/tools/bench.cpp:43-64 reads run_*(...).sim.metrics.W:
    compiled unmodified against include/ it must build and link."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "refbench"],
                   check=True)
    assert os.path.exists(REF_BENCH_BIN)


@pytest.mark.gpu
def test_reference_bench_tool_runs(binaries):
    if not os.path.exists(REF_BENCH_BIN):
        pytest.skip("oracle/_ref/ref_tools_bench not built (needs /root/reference at build time)")
    r = subprocess.run([REF_BENCH_BIN], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "MISMATCH" not in r.stdout and r.stdout.count("\n") >= 6, r.stdout

"""The reference's OWN C++ unit tests and acceptance suite (proj/tests/*.cpp),
compiled unmodified against the drop-in headers + libparplan_cuda.so by
tests/cpp/Makefile (Catch2 shim in tests/cpp/shim).  Graph and partition
tests are host-only; the cost-model, planner, oracle and acceptance suites
call build_cost_tables / ReducedGraph / plan / brute_force_plan, which run on
the B200."""
import os
import subprocess

import pytest

BUILD = os.path.join(os.path.dirname(__file__), "cpp", "_build")


def run(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (tests/cpp/Makefile needs /root/reference at build time)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=600)
    tail = "\n".join(p.stdout.splitlines()[-25:])
    assert p.returncode == 0, f"{name} failed:\n{tail}\n{p.stderr[-2000:]}"
    return p.stdout


@pytest.mark.parametrize("name", ["ref_test_graph", "ref_test_partition"])
def test_reference_host_suites(name):
    out = run(name)
    assert ", 0 failed" in out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ref_test_cost_model", "ref_test_planner", "ref_test_oracle"])
def test_reference_device_suites(name):
    out = run(name)
    assert ", 0 failed" in out


@pytest.mark.gpu
def test_reference_acceptance():
    out = run("ref_acceptance")
    assert "all criteria passed" in out

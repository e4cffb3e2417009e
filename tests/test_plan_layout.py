"""Host-only checks of the prepared plan's layout stages (csrc/plan_memory.hpp:
MemoryPlan, EffectiveSchedule) on random schedules -- tests/cpp/plan_memory_test.cpp,
compiled here with g++ (no GPU)."""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1802_04924_b200", "csrc")


def test_memory_plan_and_effective_schedule_invariants():
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "plan_memory_test")
        cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I" + CSRC,
               os.path.join(ROOT, "tests", "cpp", "plan_memory_test.cpp"), os.path.join(CSRC, "scheduler.cpp"), "-o", exe]
        b = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
        assert b.returncode == 0, b.stderr[-3000:]
        r = subprocess.run([exe, "150"], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        assert " 0 failures" in r.stdout

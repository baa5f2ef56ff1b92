"""The device-side group schedule (csrc/sched_dev.cuh: K10, and K11 behind sesgd_begin_iter_device)
is the host scheduler's (csrc/schedule.cpp, itself bit-exact with the oracle): the header is
compiled for the host with nvcc and compared for every n <= 64, every m | n, both schedules."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="needs nvcc")
def test_device_schedule_equals_host_schedule(tmp_path):
    exe = str(tmp_path / "sched_dev_check")
    subprocess.check_call(["nvcc", "-std=c++17", "-Wno-deprecated-gpu-targets", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "native", "sched_dev_check.cu"),
                           os.path.join(ROOT, "paper_2007_00433_b200", "csrc", "schedule.cpp"), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad=0" in out.stdout and "cases=" in out.stdout

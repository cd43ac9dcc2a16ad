"""CPU test of the host runtime's launch workers (csrc/launch_worker.hpp): the hand-off between
the calling thread and the per-device submit threads of a one-process communicator."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_launch_worker_handoff(tmp_path):
    exe = tmp_path / "launch_worker_stress"
    src = os.path.join(ROOT, "tests", "cpp", "launch_worker_stress.cpp")
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", src, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok:")

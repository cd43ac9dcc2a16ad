"""CPU tests of bench.py's placement: `--gpus N` is honoured or refused, never silently turned
into local mode, and a line whose n_gpus differs from --gpus is never printed."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def args(*argv):
    return bench.parse(list(argv))


def test_gpus1_is_local_mode_with_eight_ranks():
    n, devices, n_gpus, mode = bench.placement(args("--gpus", "1"), world=1, ngpu_visible=4)
    assert (n, devices, n_gpus, mode) == (8, [0] * 8, 1, "local")


def test_gpus2_without_torchrun_drives_two_devices_in_one_process():
    n, devices, n_gpus, mode = bench.placement(args("--gpus", "2"), world=1, ngpu_visible=4)
    assert mode == "one-process" and n_gpus == 2 and n == 2 and devices == [0, 1]


def test_eight_ranks_over_four_gpus_round_robin():
    n, devices, n_gpus, mode = bench.placement(args("--gpus", "4", "--ranks", "8"), world=1, ngpu_visible=4)
    assert (n, devices, n_gpus, mode) == (8, [0, 1, 2, 3, 0, 1, 2, 3], 4, "one-process")


def test_torchrun_world_must_match_gpus():
    n, devices, n_gpus, mode = bench.placement(args("--gpus", "4"), world=4, ngpu_visible=4)
    assert (n, n_gpus, mode) == (4, 4, "torchrun")
    with pytest.raises(SystemExit):
        bench.placement(args("--gpus", "8"), world=4, ngpu_visible=4)
    with pytest.raises(SystemExit):
        bench.placement(args("--gpus", "4", "--ranks", "8"), world=4, ngpu_visible=4)


def test_refuses_more_gpus_than_visible():
    with pytest.raises(SystemExit):
        bench.placement(args("--gpus", "2"), world=1, ngpu_visible=1)
    with pytest.raises(SystemExit):
        bench.placement(args("--gpus", "4", "--ranks", "2"), world=1, ngpu_visible=4)


def test_script_exits_2_without_a_line_when_gpus_unavailable():
    """On this GPU-less box `--gpus 2` must fail loudly (exit 2, empty stdout), not time local mode."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 2, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert r.stdout.strip() == ""
    assert "--gpus 2" in r.stderr


def test_reference_arm_reports_requested_gpu_count(tmp_path):
    """--impl reference at --gpus 1: n = 8 in-process ranks, n_gpus 1, JSON contract keys."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libpatsim_ref.so")):
        pytest.skip("reference library not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--chunk-bytes", "65536"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["config"]["nranks"] == 8

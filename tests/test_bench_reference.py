"""bench.py --impl reference on the CPU: the reference arm's JSON line
(metric, config, cpu_baseline with kind/cores/sample, zero-copy e2e), run
through the CLI as the driver runs it, with OMP_NUM_THREADS=1 in the
environment as torchrun sets it for its workers: the arm still uses every
host core it may run on."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_uses_all_host_cores():
    env = dict(os.environ, OMP_NUM_THREADS="1", RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--op", "dgemv",
                          "--n", "512", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] == len(os.sched_getaffinity(0)), cb
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--op", "dgemv",
                          "--n", "512", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0 and not [ln for ln in res.stdout.splitlines() if ln.startswith("{")]

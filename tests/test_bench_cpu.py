"""bench.py's host logic without a GPU: the reference arm's JSON line (the CPU oracle on a bounded
sample of the workload) and the split of per-iteration times at a breakdown event."""
import importlib.util
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench_module():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_event_split():
    b = _bench_module()
    ms = [1.0, 1.0, 1.0, 0.5, 0.5]
    # classic: entry j is iteration j + 1; an event at iteration 3 keeps iterations 1..3 as pre-event
    e = b.event_split(ms, 3, "classic")
    assert (e["n_pre"], e["n_post"]) == (3, 2)
    assert e["ms_per_iter_pre"] == pytest.approx(1.0) and e["ms_per_iter_post"] == pytest.approx(0.5)
    # SR: entry j is sweep j, so the same event leaves sweeps 0..3 pre-event
    e = b.event_split(ms, 3, "sr")
    assert (e["n_pre"], e["n_post"]) == (4, 1)
    # no event: everything is pre-event
    e = b.event_split(ms, -1, "classic")
    assert (e["n_pre"], e["n_post"], e["ms_per_iter_post"]) == (5, 0, None)
    assert b.event_split([], 2, "classic") is None


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-planes", "1"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "Gpoint-iter/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"] == "cfg3"

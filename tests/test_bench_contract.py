"""CPU: bench.py's reference arm keeps the driver's JSON-line contract (one
line, impl "reference", the GPU arm's metric / unit / direction, cpu_baseline
and a zero-copy e2e), and ranks other than 0 exit 0 without work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_built():
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    return O.ref_available()


def _bench(*args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=300,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built (make -C oracle)")
def test_reference_arm_json_line():
    lines = _bench("--impl", "reference", "--n_g", "1000000", "--steps", "3", "--warmup", "3")
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("sparsify+sync ms/iter") and "n_g=1000000" in d["metric"]
    assert d["unit"] == "ms/iter" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["ms_per_step"] == d["value"]
    assert d["warmup"] >= 5 and d["steps"] >= 3  # >= 5 warm-up steps
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "ms/iter", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["n_g"] == 1_000_000


def test_reference_arm_other_ranks_exit_without_work():
    assert _bench("--impl", "reference", "--steps", "1", "--warmup", "1",
                  env={"RANK": "1", "WORLD_SIZE": "2"}) == []

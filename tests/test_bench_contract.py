"""bench.py's reference arm on CPU (no GPU needed): the JSON line carries the
contract's keys, times the stock reference run_fixpoint on the requested K
list, and loads no repo library (its input is built on the reference side)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ref_line():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--scale", "14",
                          "--steps", "2", "--warmup", "1", "--ks", "3,kmax"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_line_contract(ref_line):
    ln = ref_line
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in ln, key
    assert ln["impl"] == "reference" and ln["unit"] == "edges/s" and ln["higher_is_better"] is True
    assert ln["e2e"]["h2d_bytes_per_step"] == 0 and ln["e2e"]["d2h_bytes_per_step"] == 0
    assert ln["cpu_baseline"]["kind"] == "reference" and ln["cpu_baseline"]["value"] == ln["value"]
    assert ln["config"]["k_values"] == [3, 79]  # s14 K_max (reference-pinned, rmat.json)
    assert ln["config"]["workload"].startswith("rmat-s14-ef16 fixpoints K=3,79")
    assert ln["steps_run"] == 2 and ln["warmup_run"] == 1


def test_reference_arm_loads_no_repo_library(ref_line):
    assert ref_line["repo_libs_loaded"] == ["oracle/_ref/libktruss_ref.so"]

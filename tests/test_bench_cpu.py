"""bench.py host logic on CPU: the reference arm derives the SAME config-2
plans as the GPU arm without importing the product package."""
import importlib.util
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_reference_plans_match_gpu_arm(reforacle):
    from paper_2504_19449_b200 import workloads as wl
    b = _bench()
    got = b.ref_config2_plans(reforacle)
    want = wl.config2_plans()
    assert len(got) == len(want) == 224
    for g, w in zip(got, want):
        assert g[0] == w[0] and g[1] == w[1] and g[2] == w[2] and g[4] == w[4]
        assert g[3] == pytest.approx(w[3], rel=0, abs=0)


def test_reference_arm_does_not_load_the_product(reforacle):
    """--impl reference runs the reference's own forward: the product library
    must not be mapped into that process."""
    code = ("import runpy, sys\nsys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0',"
            "'--ref-layers','1']\ntry:\n    runpy.run_path('bench.py', run_name='__main__')\n"
            "except SystemExit:\n    pass\n"
            "maps=open('/proc/self/maps').read()\nprint('PRODUCT_MAPPED' if 'librsparse_b200' in maps else 'CLEAN')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "CLEAN" in out.stdout and "PRODUCT_MAPPED" not in out.stdout
    import json
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["timed_seconds"] <= line["wall_seconds"]
    assert np.isfinite(line["value"]) and line["value"] > 0
    # a bounded sample (1 of 32 layers per step) is scaled to the whole stack and says so
    assert line["config"]["layers"] == 32 and line["config"]["layers_timed_per_step"] == 1
    assert "x32 from 1 to 32 layers" in line["cpu_baseline"]["sample"]
    assert line["value"] == line["cpu_baseline"]["value"] == line["e2e"]["value"]

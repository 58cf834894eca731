#!/bin/bash
# Full GPU test suite, then the bench line (with the oracle check), the
# deterministic-mode stack cost, and the reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/v_pytest.txt; tail -2 gpurun_out/v_pytest.txt
timeout 900 python bench.py --check > gpurun_out/v_bench.json 2>gpurun_out/v_bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dense --deterministic --check > gpurun_out/v_det.json 2>gpurun_out/v_det.err
python - <<'PY'
import json
for f in ("v_bench", "v_det"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), d.get("check"), d.get("speedup_vs_dense_cublas"),
              d["roofline"]["frac"], d.get("cpu_baseline", {}).get("value"))
    except Exception as e:
        print(f, "failed", e)
PY

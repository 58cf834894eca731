#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dense --deterministic --check > gpurun_out/m_det.json 2>gpurun_out/m_det.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dense --check > gpurun_out/m_fast.json 2>gpurun_out/m_fast.err
python -c "
import json
for f in ('m_det','m_fast'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['value'], d['config']['combine'], d.get('check'))"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m_ref.json 2>gpurun_out/m_ref.err
python -c "
import json
d=json.load(open('gpurun_out/m_ref.json')); print('ref', d['value'], d['timed_seconds'], d['wall_seconds'], d['host'].get('MemAvailable'))"

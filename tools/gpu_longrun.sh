#!/bin/bash
# Long runs: 20000 consecutive tokens through the stack (and through the cross-process exchange
# path at world size 1), then the oracle check of the last outputs -- counters, epochs and the
# double-buffered t state must not drift over many launches.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20000 --warmup 5 --no-cpu --no-dense --check > gpurun_out/long_stack.json 2> gpurun_out/long_stack.err
python -c "import json;d=json.loads(open('gpurun_out/long_stack.json').read().strip().splitlines()[-1]);print('stack', d['steps'], round(d['value'],1), d['config']['step_ms_p10_p50_p90'], d['check'], d['clocks'])"
timeout 900 python bench.py --steps 20000 --warmup 5 --no-cpu --no-dense --check --force-sharded --exchange kernel > gpurun_out/long_peer.json 2> gpurun_out/long_peer.err
python -c "import json;d=json.loads(open('gpurun_out/long_peer.json').read().strip().splitlines()[-1]);print('peer', d['steps'], round(d['value'],1), d['config']['step_ms_p10_p50_p90'], d['check'])"

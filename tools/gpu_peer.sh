#!/bin/bash
# The cross-process exchange path at world size 1 (tests + bench), plus the default bench A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_config2.py -m gpu -q -p no:cacheprovider > gpurun_out/peer_pytest.txt 2>&1
tail -3 gpurun_out/peer_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dense --check --force-sharded --exchange kernel > gpurun_out/peer_bench.json 2> gpurun_out/peer_bench.err
python -c "import json;d=json.loads(open('gpurun_out/peer_bench.json').read().strip().splitlines()[-1]);print('peer', round(d['value'],1), d['e2e']['value'], d.get('check'), d['config']['parallelism'])" 2>&1 | tail -2
tail -3 gpurun_out/peer_bench.err
for rep in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense --check > gpurun_out/peer_default_$rep.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/peer_default_$rep.json').read().strip().splitlines()[-1]);print('default', round(d['value'],1), d['check']['ok'])" 2>&1 | tail -1
done

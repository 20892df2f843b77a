#!/bin/bash
# Same-box A/B of the C2 end-to-end leg over pack-thread counts (value + e2e)
for i in 1 2; do for T in "$@"; do
  timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-fault --pack-threads $T \
    > gpurun_out/e2e_$T.json 2> gpurun_out/e2e_$T.err
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$T.json').read().strip().splitlines()[-1]); print('pack', $T, d['value'], d['e2e']['value'], d['e2e'].get('host_ms_per_step'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/e2e_$T.err
done; done
nproc

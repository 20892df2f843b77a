#!/bin/bash
# Replica-parallel repeatability: N = 2 and N = 4 on one box, twice each.
mkdir -p gpurun_out
for i in 1 2; do for np in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $np \
    --mode replica --steps 30 --warmup 5 --no-cpu-baseline --no-fault --quick \
    > gpurun_out/rr_${np}_${i}.json 2> gpurun_out/rr_${np}_$i.err
  python -c "import json; d=json.loads(open('gpurun_out/rr_${np}_${i}.json').read().strip().splitlines()[-1]); print($np, $i, d['value'], d['ms_per_step'], d['roofline']['other_ms_per_step'])"
done; done

#!/bin/bash
# Group-per-GPU weak scaling with the driver's command shape: N = 1, 2, 4.
mkdir -p gpurun_out
for np in 1 2 4; do
  if [ $np = 1 ]; then
    timeout 600 python bench.py --gpus 1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/scale_$np.json 2> gpurun_out/scale_$np.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 500)) bench.py --gpus $np --steps 30 --warmup 5 --no-cpu-baseline \
      > gpurun_out/scale_$np.json 2> gpurun_out/scale_$np.err
  fi
  python -c "import json; d=json.loads(open('gpurun_out/scale_$np.json').read().strip().splitlines()[-1]); print($np, d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
done

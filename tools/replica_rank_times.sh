for i in 1 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus 4 \
    --mode replica --steps 30 --warmup 5 --no-cpu-baseline --no-fault --quick \
    > gpurun_out/rr4_$i.json 2> gpurun_out/rr4_$i.err
  grep "per-rank" gpurun_out/rr4_$i.err
done

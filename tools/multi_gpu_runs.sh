#!/bin/bash
# Multi-GPU measurement batch (run under gpurun --gpus N): NCCL parity tests,
# replica-parallel C2 at 2 and N GPUs, an 8-replica group at 2 per rank, C4 over
# NCCL, and the group-per-GPU (weak scaling) line. Outputs under gpurun_out/.
N=${1:-4}
TAG=${2:-r2_g$N}
mkdir -p gpurun_out
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $np "$@" \
    > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err
  echo "$name rc=$? $(tail -c 300 gpurun_out/${TAG}_$name.json)"
}
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/${TAG}_dist_tests.log 2>&1
tail -2 gpurun_out/${TAG}_dist_tests.log
run replica_n2 2 --mode replica --steps 30 --warmup 5 --no-cpu-baseline --no-fault
run replica_n$N $N --mode replica --steps 30 --warmup 5 --no-cpu-baseline --no-fault
run replica_n${N}_r8 $N --mode replica --replicas-dist 8 --steps 30 --warmup 5 --no-cpu-baseline --no-fault
run c4_n$N $N --workload c4 --steps 12 --warmup 3
run group_n$N $N --steps 30 --warmup 5 --no-cpu-baseline

set -x
timeout 600 python bench.py > gpurun_out/r_n1.json 2>gpurun_out/r_n1.err
for N in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/r_n$N.json 2>gpurun_out/r_n$N.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --mode replica > gpurun_out/r_rep2.json 2>gpurun_out/r_rep2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --mode replica > gpurun_out/r_rep4.json 2>gpurun_out/r_rep4.err
timeout 600 python bench.py --workload c3 > gpurun_out/r_c3.json 2>gpurun_out/r_c3.err
timeout 600 python bench.py --workload c5 > gpurun_out/r_c5.json 2>gpurun_out/r_c5.err
for N in 1 2 4; do if [ $N = 1 ]; then timeout 600 python bench.py --workload c4 > gpurun_out/r_c4_n1.json 2>gpurun_out/r_c4_n1.err; else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --workload c4 > gpurun_out/r_c4_n$N.json 2>gpurun_out/r_c4_n$N.err; fi; done
ls -la gpurun_out/r_*.json

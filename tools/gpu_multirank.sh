export MTNN_BENCH_SHARE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 1 --exp-max 11 --no-e2e --no-cpu > gpurun_out/mr_sweep.json 2> gpurun_out/mr_sweep.err; echo rc=$?; tail -3 gpurun_out/mr_sweep.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --workload large --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/mr_large.json 2> gpurun_out/mr_large.err; echo rc=$?; tail -3 gpurun_out/mr_large.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --workload fcn --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/mr_fcn.json 2> gpurun_out/mr_fcn.err; echo rc=$?; tail -3 gpurun_out/mr_fcn.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo rc=$?
cat gpurun_out/mr_*.json | cut -c1-300

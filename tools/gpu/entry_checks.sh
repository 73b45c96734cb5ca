mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-louvain > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo "rc=$?" >> gpurun_out/torchrun1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun1_ref.json 2> gpurun_out/torchrun1_ref.err; echo "rc=$?" >> gpurun_out/torchrun1_ref.err

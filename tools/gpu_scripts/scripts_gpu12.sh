nvidia-smi topo -m > gpurun_out/topo2.txt 2>&1
python -m pytest tests/test_gpu_railowner.py -q --timeout 600 -rf > gpurun_out/gpu_railowner.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/ref_n2.json 2> gpurun_out/ref_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/railowner_bench.py --units 8 > gpurun_out/railowner_n2.json 2> gpurun_out/railowner_n2.err
echo finished

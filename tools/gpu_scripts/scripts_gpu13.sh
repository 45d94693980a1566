timeout 600 python -m pytest tests/test_gpu_railowner.py -q --timeout 300 -rf -x > gpurun_out/gpu_railowner2.log 2>&1; echo "railowner rc=$?" >> gpurun_out/rc13.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_n2a.json 2> gpurun_out/bench_n2a.err; echo "bench_noe2e rc=$?" >> gpurun_out/rc13.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2b.json 2> gpurun_out/bench_n2b.err; echo "bench rc=$?" >> gpurun_out/rc13.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 tools/railowner_bench.py --units 8 > gpurun_out/railowner_n2b.json 2> gpurun_out/railowner_n2b.err; echo "ro_bench rc=$?" >> gpurun_out/rc13.txt
free -g >> gpurun_out/rc13.txt
echo finished

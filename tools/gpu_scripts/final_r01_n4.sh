# Round-closing multi-GPU confirmation: -m gpu suite on 4 GPUs (multi-rank cases run), N=2 and N=4 bench lines.
python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/final4_gpu_tests.log 2>&1; echo "tests rc=$?" > gpurun_out/final4_rc.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/final_bench_n2.json 2> gpurun_out/final_bench_n2.err; echo "bench2 rc=$?" >> gpurun_out/final4_rc.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/final_bench_n4.json 2> gpurun_out/final_bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/final4_rc.txt
echo finished

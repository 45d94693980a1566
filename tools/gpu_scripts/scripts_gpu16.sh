python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests16.log 2>&1; echo "tests rc=$?" > gpurun_out/rc16.txt
RAILS_HIST_IMPL=3 python -m pytest tests -m gpu -q --timeout 600 -rf -k "histogram or c1 or pack or determinism or combine" > gpurun_out/gpu_tests16_w1.log 2>&1; echo "w1 rc=$?" >> gpurun_out/rc16.txt
python tools/kernel_bench.py --only hist --out gpurun_out/kernels_v11.json > gpurun_out/kb16.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/rc16.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 tools/railowner_bench.py --units 8 > gpurun_out/railowner_n4.json 2> gpurun_out/railowner_n4.err; echo "ro4 rc=$?" >> gpurun_out/rc16.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/ref_n4.json 2> gpurun_out/ref_n4.err; echo "ref4 rc=$?" >> gpurun_out/rc16.txt
echo finished

python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests5.log 2>&1
python tools/kernel_bench.py --out gpurun_out/kernels_new.json > gpurun_out/kb3.log 2>&1
RAILS_CHAIN_IMPL=1 python tools/kernel_bench.py --only c2,c5 --out gpurun_out/kernels_warpchain.json > gpurun_out/kb4.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo finished

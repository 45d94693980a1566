python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/gpu_tests9.log 2>&1
RAILS_HIST_IMPL=2 python -m pytest tests -m gpu -q --timeout 600 -rf -k "histogram or c1" > gpurun_out/gpu_tests9_h2.log 2>&1
python tools/kernel_bench.py --only pack,hist --out gpurun_out/kernels_v6.json > gpurun_out/kb9.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
echo finished

python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/gpu_tests11.log 2>&1
RAILS_HIST_IMPL=3 python -m pytest tests -m gpu -q --timeout 600 -rf -k "histogram or c1 or pack or determinism" > gpurun_out/gpu_tests11_w1.log 2>&1
python tools/kernel_bench.py --only pack,hist --out gpurun_out/kernels_v8.json > gpurun_out/kb11.log 2>&1
echo finished

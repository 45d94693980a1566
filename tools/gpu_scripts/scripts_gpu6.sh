python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests6.log 2>&1
python tools/kernel_bench.py --out gpurun_out/kernels_v3.json > gpurun_out/kb6.log 2>&1
echo finished

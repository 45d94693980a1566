python -m pytest tests -m gpu -q --timeout 600 -rf -k "pack or c4 or smoke" > gpurun_out/gpu_tests3.log 2>&1
RAILS_PACK_IMPL=2 python -m pytest tests -m gpu -q --timeout 600 -rf -k "pack or c1 or c3 or determinism" > gpurun_out/gpu_tests3_tma.log 2>&1
python tools/kernel_bench.py --out gpurun_out/kernels_r01.json > gpurun_out/kb.log 2>&1
echo finished

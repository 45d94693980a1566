python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests18.log 2>&1; echo "tests rc=$?" > gpurun_out/rc18.txt
RAILS_CHAIN_IMPL=1 python -m pytest tests -m gpu -q --timeout 600 -rf -k "schedule or c2 or lpt or c1" > gpurun_out/gpu_tests18_warp.log 2>&1; echo "warpchain rc=$?" >> gpurun_out/rc18.txt
python tools/kernel_bench.py --out gpurun_out/kernels_v13.json > gpurun_out/kb18.log 2>&1; echo "kb rc=$?" >> gpurun_out/rc18.txt
echo finished

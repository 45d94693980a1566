python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests19.log 2>&1; echo "tests rc=$?" > gpurun_out/rc19.txt
python tools/kernel_bench.py --only pack,hist,c2,c5 --out gpurun_out/kernels_v14.json > gpurun_out/kb19.log 2>&1; echo "kb rc=$?" >> gpurun_out/rc19.txt
echo finished

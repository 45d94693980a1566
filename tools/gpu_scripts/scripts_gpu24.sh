python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests24.log 2>&1; echo "tests rc=$?" > gpurun_out/rc24.txt
python tools/kernel_bench.py --only hist,c2,c5 --out gpurun_out/kernels_v15.json > gpurun_out/kb24.log 2>&1; echo "kb rc=$?" >> gpurun_out/rc24.txt
echo finished

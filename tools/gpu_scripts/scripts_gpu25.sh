python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests25.log 2>&1; echo "tests rc=$?" > gpurun_out/rc25.txt
python tools/kernel_bench.py --out gpurun_out/kernels_v16.json > gpurun_out/kb25.log 2>&1; echo "kb rc=$?" >> gpurun_out/rc25.txt
python bench.py --steps 20 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc=$?" >> gpurun_out/rc25.txt
echo finished

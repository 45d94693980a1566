python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests7.log 2>&1
python tools/kernel_bench.py --out gpurun_out/kernels_v4.json > gpurun_out/kb7.log 2>&1
python tools/kernel_bench.py --only c2,c5 > gpurun_out/kb7b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_c2c5.csv python tools/kernel_bench.py --only c2,c5 > gpurun_out/ncu7.log 2>&1
echo finished

python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests15.log 2>&1
python tools/kernel_bench.py --only c2,c5 --out gpurun_out/kernels_v10.json > gpurun_out/kb15.log 2>&1
python tools/kernel_bench.py --only c2 > gpurun_out/kb15b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_c2_v2.csv python tools/kernel_bench.py --only c2 > gpurun_out/ncu15.log 2>&1
echo finished

python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/gpu_tests10.log 2>&1
RAILS_HIST_IMPL=3 python -m pytest tests -m gpu -q --timeout 600 -rf -k "histogram or c1 or pack or determinism" > gpurun_out/gpu_tests10_w1.log 2>&1
python tools/kernel_bench.py --only pack,hist --out gpurun_out/kernels_v7.json > gpurun_out/kb10.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hist_w1" -s 3 -c 1 -o gpurun_out/prof_hist_w1 python tools/kernel_bench.py --only pack,hist > gpurun_out/ncu10.log 2>&1
echo finished

python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests8.log 2>&1
RAILS_HIST_IMPL=1 python -m pytest tests -m gpu -q --timeout 600 -rf -k "histogram or c1 or pack" > gpurun_out/gpu_tests8_oldhist.log 2>&1
python tools/kernel_bench.py --only hist --out gpurun_out/kernels_v5.json > gpurun_out/kb8.log 2>&1
python tools/kernel_bench.py --only hist > gpurun_out/kb8b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hist_rank2" -s 3 -c 1 -o gpurun_out/prof_hist3 python tools/kernel_bench.py --only hist > gpurun_out/ncu8.log 2>&1
echo finished

python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests4.log 2>&1
RAILS_CHAIN_IMPL=1 python -m pytest tests -m gpu -q --timeout 600 -rf -k "schedule or c2" > gpurun_out/gpu_tests4_warpchain.log 2>&1
python tools/kernel_bench.py --only hist,c2,c5 --out gpurun_out/kernels_r01b.json > gpurun_out/kb2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hist_rank|k_eval_node|k_lpt_thread|k_chunk_sort" -c 4 -o gpurun_out/prof_sched python tools/kernel_bench.py --only hist,c2,c5 > gpurun_out/ncu_sched.log 2>&1
echo finished

python tools/kernel_bench.py --only pack,hist > gpurun_out/kb5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_chunk_sort|k_lpt_thread|k_eval_node2" -c 3 -o gpurun_out/prof_c3sched python tools/kernel_bench.py --only pack,hist > gpurun_out/ncu5a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hist_rank" -s 16 -c 1 -o gpurun_out/prof_hist2 python tools/kernel_bench.py --only pack,hist > gpurun_out/ncu5b.log 2>&1
echo finished

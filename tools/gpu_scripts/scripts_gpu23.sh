python tools/combine_bench.py --out gpurun_out/combine_r01.json > gpurun_out/combine.log 2>&1; echo "combine rc=$?" > gpurun_out/rc23.txt
python tools/kernel_bench.py --only hist > gpurun_out/kb23.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_chunk_sort|k_lpt_thread" -c 2 -o gpurun_out/prof_c4sched python tools/kernel_bench.py --only hist > gpurun_out/ncu23.log 2>&1
echo finished

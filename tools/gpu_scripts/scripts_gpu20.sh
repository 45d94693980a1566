python tools/kernel_bench.py --only pack,hist > gpurun_out/kb20.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_chunk|k_lpt|k_expand|k_hist|k_eval" --csv --log-file gpurun_out/launches_sched.csv python tools/kernel_bench.py --only pack,hist > gpurun_out/ncu20.log 2>&1
python tools/combine_bench.py --out gpurun_out/combine_r01.json > gpurun_out/combine.log 2>&1; echo "combine rc=$?" > gpurun_out/rc20.txt
echo finished

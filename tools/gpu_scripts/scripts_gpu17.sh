python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests17.log 2>&1; echo "tests rc=$?" > gpurun_out/rc17.txt
python tools/kernel_bench.py --out gpurun_out/kernels_v12.json > gpurun_out/kb17.log 2>&1; echo "kb rc=$?" >> gpurun_out/rc17.txt
python tools/kernel_bench.py --only hist > gpurun_out/kb17h.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_hist_w1 -s 3 -c 1 -o gpurun_out/prof_hist_final python tools/kernel_bench.py --only hist > gpurun_out/ncu17a.log 2>&1
python tools/kernel_bench.py --only c2 > gpurun_out/kb17c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_chunk_sort|k_lpt|k_eval_node2" -c 3 -o gpurun_out/prof_sched_c2 python tools/kernel_bench.py --only c2 > gpurun_out/ncu17b.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?" >> gpurun_out/rc17.txt
echo finished

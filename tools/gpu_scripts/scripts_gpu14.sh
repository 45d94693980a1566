python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/gpu_tests14.log 2>&1
python tools/kernel_bench.py --only pack,hist --out gpurun_out/kernels_v9.json > gpurun_out/kb14.log 2>&1
python tools/policy_report.py --out gpurun_out/policy_r01.json > gpurun_out/policy.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_full.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_pack -s 3 -c 1 --csv --log-file gpurun_out/pack_traffic_full.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu14.log 2>&1
echo finished

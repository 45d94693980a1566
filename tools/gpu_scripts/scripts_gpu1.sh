set -x
python -m pytest tests -m gpu -q --timeout 600 -rf -k "c4 or c3 or report" -s > gpurun_out/gpu_tests2.log 2>&1
nvidia-smi > gpurun_out/nvsmi.txt; free -g >> gpurun_out/nvsmi.txt; nproc >> gpurun_out/nvsmi.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --nd 8 > gpurun_out/plain_nd8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pack -s 3 -c 1 -o gpurun_out/prof_pack python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --nd 8 > gpurun_out/ncu_pack.log 2>&1
echo finished
